/*
 * moe.h -- C ABI of the B200-native expert-parallel MoE layer (libmoe.so).
 *
 * The hot path of arxiv 2605.05049 ("Piper"): one MoE layer under expert
 * parallelism ("expert data parallelism"; PAPER.md:351-365
 * dispatch/combine all-to-alls), forward and backward, on 1/2/4/8 B200s of one
 * NVSwitch box.  Step names follow SURVEY.md §8(a): F0 router logits, F1 route,
 * F2 permute, F3 dispatch, F4 expert FFN, F5 combine, F6 unpermute, and the
 * backward twins B0..B6.  Symbols follow PAPER.md Table II.
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Pointers named x, w_*, logits, ... are DEVICE pointers on the ctx's device;
 *   `stream` is a cudaStream_t (0 = legacy default stream).  Every call is
 *   stream-ordered and asynchronous: the returned status covers host-side
 *   validation and launch only.  A receive overflow sets a device error word read by
 *   moe_ctx_get_device_error().  A peer flag that never arrives (10 s) records
 *   MOE_ERR_TIMEOUT in that word and then TRAPS the kernel: the fault is sticky, so the
 *   process's next synchronising CUDA call fails (MOE_ERR_CUDA from libmoe) rather than
 *   later calls silently running on an incomplete receive buffer.
 * - The caller owns every buffer.  Buffers that a PEER writes into (the
 *   destinations of the four all-to-alls: xr, ys, dout_r, dxs) must come from
 *   moe_symm_alloc(); otherwise the call returns MOE_ERR_NOT_SYMMETRIC.
 * - Validation happens before any launch: MOE_ERR_INVALID_ARG for ep_size not in
 *   {1,2,4,8}, EP does not divide E, k < 1 or k > E,
 *   ep_rank outside [0,EP), d or f not a multiple of 64 (TMA/UMMA K-blocks of 64
 *   bf16; the grouped FFN also needs f % 128 == 0 -- narrower than the survey's d % 8,
 *   f % 16, a deliberate choice: every contraction runs whole 64-wide K-blocks), k > 32,
 *   E > 256, T_local < 0, or a NULL required pointer.  T_local = 0 is legal; the
 *   collective calls still take part in the exchange.
 * - Collective calls (moe_dispatch, moe_dispatch_bwd, moe_combine,
 *   moe_combine_bwd, their _range variants, the fused *_combine / *_dispatch FFN
 *   calls, moe_dispatch_expert_ffn_up, moe_combine_bwd_expert_ffn_dh, the moe_dedup_*
 *   all-to-alls, moe_migrate, moe_all_to_all, moe_symm_alloc) must be issued by every EP
 *   rank in the same order, like NCCL collectives.  Not thread-safe; one ctx per
 *   (process, GPU, layer activation context) -- several ctxs per process are fine
 *   (the PP x EP executor keeps one per layer and in-flight micro-batch).
 * - A collective's destination buffer is written by PEERS from the moment they enter
 *   the call: a rank must not write it itself (e.g. zero it) after its previous
 *   collective returned unless every rank has passed that point (a barrier), or the
 *   peers' rows can be overwritten.  The layer never writes them locally.
 * - The collectives' epoch counter lives in device memory and is advanced by the
 *   kernels, so a sequence of calls may be captured once in a CUDA graph and replayed.
 * - Determinism: identical inputs give bit-identical outputs on every call (no
 *   float atomics, fixed reduction orders); buffers may be reused across calls.
 * - Dtypes: bf16 activations/weights/messages (moe_bf16 = raw bf16 bits), fp32
 *   logits/gates/weight gradients, int32 indices and counts.
 *
 * Layouts
 * -------
 * Expert weights, K-major ("transposed") for the tensor cores:
 *   w_gu   [G, 2f, d]  rows 0..f-1 = W_gate^T, rows f..2f-1 = W_up^T
 *   w_down [G, d, f]   = W_down^T
 *   w_r    [E, d]      = W_r^T (router)
 * Send layout (per source rank): rows of xs/ys/dxs are grouped by global
 *   expert e; expert e's kept rows occupy [off[e], off[e]+counts[e]) with
 *   off = exclusive scan of counts; inside an expert, rows are in assignment
 *   order a = j*T_local + t (reading R5, slot-major).
 * Receive layout (per owner rank): local expert e_l (global e = ep_rank*E_l+e_l)
 *   owns the segment [seg_base[e_l], seg_base[e_l+1]), seg_base[0] = 0,
 *   seg_base[e_l+1] = seg_base[e_l] + roundup(expert_rows[e_l], MOE_ALIGN_ROWS).
 *   Inside a segment rows are ordered (source rank r, position p); rows past
 *   expert_rows[e_l] are padding and are ZERO in xr and dout_r after the
 *   transfer (reading R7; the padding makes every expert a whole number of
 *   128-row UMMA tiles).
 * Layout record (int32, moe_layout_ints() entries, written by moe_dispatch):
 *   [MOE_LAYOUT_COUNTS_ALL  .. +EP*E)   counts_all[r][e]  kept rows from source r to expert e
 *   [MOE_LAYOUT_EXPERT_ROWS .. +E_l)    expert_rows[e_l]  rows received by local expert e_l
 *   [MOE_LAYOUT_SEG_BASE    .. +E_l+1)  seg_base[e_l]     segment starts (see above)
 */
#ifndef MOE_H_
#define MOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef uint16_t moe_bf16;       /* raw bfloat16 bits */
typedef void* moe_stream;        /* cudaStream_t */

#define MOE_ALIGN_ROWS 128       /* receive-segment alignment (rows) */
#define MOE_IPC_HANDLE_BYTES 64  /* size of one exported symmetric-heap handle */
#define MOE_MAX_EP 8

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARG = 1,
  MOE_ERR_CUDA = 2,
  MOE_ERR_NOT_SYMMETRIC = 3,   /* all-to-all destination not from moe_symm_alloc */
  MOE_ERR_OUT_OF_MEMORY = 4,   /* symmetric heap exhausted */
  MOE_ERR_RECV_OVERFLOW = 5,   /* device-side: receive rows beyond the buffer */
  MOE_ERR_TIMEOUT = 6,         /* device-side: a peer flag never arrived (10 s; the kernel traps) */
  MOE_ERR_NOT_READY = 7        /* collective call before moe_ctx_open_peers */
} moe_status;

enum { MOE_LAYOUT_COUNTS_ALL = 0, MOE_LAYOUT_EXPERT_ROWS = 1, MOE_LAYOUT_SEG_BASE = 2 };

/* Problem statement, Table II symbols + the capacity factor. */
typedef struct {
  int64_t T_local;          /* T_r = b*s/EP tokens on this rank (reading R10) */
  int32_t d;                /* hidden size d_model */
  int32_t E;                /* routed experts */
  int32_t k;                /* top-k */
  int32_t f;                /* expert FFN width d_ffn^MoE */
  int32_t E_shared;         /* E_s always-active shared experts (width f each; local) */
  float capacity_factor;    /* cf > 0: C = ceil(cf*k*T_local/E) per (source, expert); cf <= 0: dropless */
  int32_t ep_size;          /* EP degree (1, 2, 4 or 8) */
  int32_t ep_rank;          /* rank in the EP group */
} moe_shape;

typedef struct moe_ctx moe_ctx;   /* opaque: symmetric heap, peer table, flags, scratch */
/* No moe_ctx_attach_nccl (SURVEY.md §8(b) listed it "baseline only"): libmoe has no NCCL
 * dependency; the NCCL baselines (bench.py --a2a) run through torch.distributed beside it. */

/* ---------------- context ---------------- */

/* Creates a ctx on `device` and allocates its symmetric heap of `symm_heap_bytes`
 * (plus an internal region for the count matrix and flags).  EP=1 needs no peers. */
moe_status moe_ctx_create(moe_ctx** ctx, const moe_shape* shape, int device, size_t symm_heap_bytes);
/* Writes MOE_IPC_HANDLE_BYTES bytes identifying this rank's heap (cudaIpcMemHandle). */
moe_status moe_ctx_export_handle(moe_ctx* ctx, void* handle_out);
/* handles = ep_size * MOE_IPC_HANDLE_BYTES bytes in rank order (all-gathered by the
 * caller, e.g. over torch.distributed); maps every peer's heap.  Collective. */
moe_status moe_ctx_open_peers(moe_ctx* ctx, const void* handles);
/* Bump allocation from the symmetric heap, 256-byte aligned.  Collective: every rank
 * must request the same sizes in the same order so offsets agree. */
moe_status moe_symm_alloc(moe_ctx* ctx, size_t bytes, void** ptr);
/* Releases the LAST symmetric allocation (LIFO, like the bump allocator it undoes);
 * MOE_ERR_INVALID_ARG for any other pointer.  Collective, like moe_symm_alloc. */
moe_status moe_symm_free(moe_ctx* ctx, void* ptr);
/* FNV-1a fingerprint of this rank's (offset, size) allocation sequence.  Peers write into a
 * symmetric buffer at ITS offset in every heap, so every rank must have made the same
 * allocations in the same order: all-gather the fingerprints (like the IPC handles) and pass
 * them, in rank order, to moe_ctx_verify_symmetric, which returns MOE_ERR_NOT_SYMMETRIC when
 * any rank's sequence differs from this one.  Collective calls additionally check, on every
 * call, that their destination range [ptr, ptr + required bytes) lies inside ONE allocation
 * (required = recv_rows_max x d x 2 for xr / dout_r, T_local x k x d x 2 for ys / dxs, the
 * dedup bounds for the moe_dedup_* buffers). */
moe_status moe_symm_fingerprint(moe_ctx* ctx, uint64_t* out);
/* Device memory held by the ctx (any pointer may be NULL): the symmetric heap's size and the
 * bytes allocated from it so far, and the total of every device allocation the ctx made
 * (heap + scratch).  Host-only; used for the per-stage memory account of the PP x EP executor
 * against PAPER.md Eq. 4 (1F1B per-stage memory). */
moe_status moe_ctx_device_bytes(moe_ctx* ctx, size_t* heap_bytes, size_t* heap_used,
                                size_t* total_bytes);
moe_status moe_ctx_verify_symmetric(moe_ctx* ctx, const uint64_t* fingerprints);
/* Expert placement (SURVEY.md §8(f) NEXT-2 expert migration, §VI): placement[e] =
 * global slot of expert e (host int32 [E], a permutation of [0, E)); expert e then lives on
 * rank placement[e] / E_l in local slot placement[e] % E_l, and every receive layout, GEMM
 * group g (= local slot) and weight index w_gu[g], w_down[g] refers to slots.  Default: the
 * identity (contiguous ownership).  Collective: every rank sets the same placement; it
 * synchronises the device.  MOE_ERR_INVALID_ARG if not a permutation. */
moe_status moe_ctx_set_placement(moe_ctx* ctx, const int32_t* placement);
/* Equal-split all-to-all over the peer maps (BASELINE.json config 5, the sweep against
 * ncclAllToAll; SPEC.md:476 transpose law): send = [EP][bytes_per_peer] bytes (device, local),
 * recv = [EP][bytes_per_peer] SYMMETRIC; chunk q of send lands in chunk `ep_rank` of rank q's
 * recv.  The layout is static, so one launch does the stores and the completion flags (no
 * counts round); returns (stream-ordered) when this rank's recv is complete.  Collective.
 * bytes_per_peer % 16 == 0; 0 is a no-op. */
moe_status moe_all_to_all(moe_ctx* ctx, const void* send, void* recv, size_t bytes_per_peer,
                          moe_stream stream);
/* Migration trigger (an external scheduler "inspects the growing load
 * imbalance, and whenever it crosses a pre-determined threshold" runs Alg. 2; reading R20):
 * *out = max_q s_q / mean_q s_q, s_q = sum of loads[e] over the experts placement puts on
 * rank q (1.0 when every load is 0).  Host-only, deterministic. */
moe_status moe_load_imbalance(const int64_t* loads, const int32_t* placement, int32_t E,
                              int32_t ep, double* out);
/* Alg. 2 of PAPER.md:672-706 (hill-climbing swap-based minimal rebalancing) on host data:
 * groups = the EP owners' slots, item loads = loads[e] (e.g. the routed rows per expert from
 * the layout record); at most max_iters (paper: T = 100) iterations, each swapping the pair
 * of experts between the most- and least-loaded ranks that reduces their difference most
 * (ties: lowest index).  placement (host [E]) is updated in place; n_swaps = swaps applied.
 * Deterministic: every rank computes the same result from the same loads. */
moe_status moe_rebalance(const int64_t* loads, int32_t E, int32_t ep, int32_t max_iters,
                         int32_t* placement, int32_t* n_swaps);
/* Expert migration transfer (NEXT-2; "migrate experts" whenever the imbalance
 * crosses a threshold; Table PAPER.md:650-668 costs 48 d f bytes of state per expert; reading
 * R17).  Collective over the EP group: every rank passes the same old_placement and
 * new_placement (host int32 [E], expert -> global slot, permutations of [0, E)).
 * src, dst: SYMMETRIC buffers (moe_symm_alloc, the same offset on every rank, each
 * [E_l][bytes_per_expert] bytes, not overlapping).  src holds this rank's experts' state in
 * the OLD placement's local-slot order; on return (stream-ordered) dst holds the state of the
 * experts new_placement assigns to this rank, in the NEW local-slot order.  Each expert is
 * pushed by its old owner straight into its new owner's dst over NVSwitch (local slot moves
 * are local copies); one launch: a device barrier first (every rank has reached the call, so
 * no peer is still reading its dst from earlier stream work), then the stores, then the
 * completion flags.  Call once per state tensor (weights, weight gradients, optimizer state).
 * It does NOT switch the ctx's placement: call moe_ctx_set_placement(new_placement) after the
 * last state tensor has moved.  MOE_ERR_INVALID_ARG: not permutations, bytes_per_expert not a
 * positive multiple of 16, E_l > 256; MOE_ERR_NOT_SYMMETRIC: src or dst range outside the
 * symmetric heap's allocations. */
moe_status moe_migrate(moe_ctx* ctx, const int32_t* old_placement, const int32_t* new_placement,
                       const void* src, void* dst, size_t bytes_per_expert, moe_stream stream);
/* SM budgets for the calls issued after it (0 = all SMs): grouped-GEMM launches use at most
 * gemm_sms SMs and all-to-all transfer launches 2 blocks on each of comm_sms SMs, so that a
 * GEMM and a transfer issued on two streams run concurrently on disjoint SMs (used to overlap
 * the shared-expert GEMMs with dispatch / combine_bwd).  The GEMM
 * launches that carry a transfer (moe_dispatch_expert_ffn_up, moe_combine_bwd_expert_ffn_dh)
 * use gemm_sms SMs if it is set, else comm_sms. */
moe_status moe_ctx_set_sm_limits(moe_ctx* ctx, int gemm_sms, int comm_sms);
/* Synchronises the device; returns MOE_OK or the first device-side error recorded. */
moe_status moe_ctx_get_device_error(moe_ctx* ctx);
moe_status moe_ctx_destroy(moe_ctx* ctx);
const char* moe_status_string(moe_status status);

/* Derived sizes (host-only; no ctx needed). */
int64_t moe_capacity(const moe_shape* shape);        /* C, or -1 when dropless */
int64_t moe_recv_rows_max(const moe_shape* shape);   /* rows to allocate for xr / dout_r / dxr */
int64_t moe_layout_ints(const moe_shape* shape);     /* int32 entries of a layout record */
int64_t moe_layout_offset(const moe_shape* shape, int field);

/* ---------------- F0 / B0 router ("routing") ---------------- */

/* logits[t,e] = sum_c x[t,c] w_r[e,c] (+ bias[e]); bf16 x bf16 -> fp32 on the tensor
 * cores.  x [T_local,d], w_r [E,d], bias [E] fp32 or NULL, logits [T_local,E] fp32. */
moe_status moe_router_logits(moe_ctx* ctx, const moe_bf16* x, const moe_bf16* w_r,
                             const float* bias_or_null, float* logits, moe_stream stream);
/* dx_router[t,c] = sum_e dlogits[t,e] w_r[e,c]   (fp32 [T_local,d], overwritten);
 * dw_r[e,c] (+)= sum_t dlogits[t,e] x[t,c]       (fp32 [E,d]; accumulate != 0 adds). */
moe_status moe_router_logits_bwd(moe_ctx* ctx, const moe_bf16* x, const moe_bf16* w_r,
                                 const float* dlogits, float* dx_router, float* dw_r,
                                 int accumulate, moe_stream stream);

/* ---------------- F1 / B1 route: top-k gating ---------------- */

/* Per token: the k largest fp32 logits ordered by descending value, ties to the lower
 * expert index (-0.0 == +0.0, NaN below -inf; readings R2, R3); gates = softmax over
 * the k selected logits (k > 1) or the full-softmax probability of the top expert
 * (k = 1) (reading R1).  logits [T_local,E] -> topk_idx [T_local,k] int32,
 * gates [T_local,k] fp32.  Indices are bit-exact functions of the logits. */
moe_status moe_route(moe_ctx* ctx, const float* logits, int32_t* topk_idx, float* gates,
                     moe_stream stream);
/* dlogits[t,e_j] = g_j (dg_j - sum_i g_i dg_i), zero elsewhere (k > 1); k = 1 uses the
 * full softmax and reads `logits` (may be NULL when k > 1).  dlogits [T_local,E] fp32. */
moe_status moe_route_bwd(moe_ctx* ctx, const float* logits, const int32_t* topk_idx,
                         const float* gates, const float* dgates, float* dlogits,
                         moe_stream stream);

/* ---------------- F2 / B2 permute (PAPER.md:129 token dropping, 231 s_e) ---------------- */

/* Histogram, scan, capacity and scatter, per source rank (readings R4, R5):
 * p(t,j) = #earlier assignments a' < a = j*T_local+t on the same expert; kept iff
 * p < C; counts[e] = #kept; dest_row[t,j] = off[e] + p or -1 (dropped);
 * xs[dest_row[t,j]] = x[t] (bit copy).  counts [E] int32, dest_row [T_local,k] int32,
 * xs [T_local*k, d] bf16 (rows [0, sum counts) written; NULL = indices only). */
moe_status moe_permute(moe_ctx* ctx, const moe_bf16* x, const int32_t* topk_idx,
                       int32_t* counts, int32_t* dest_row, moe_bf16* xs, moe_stream stream);
/* F2 + F3 at EP = 1 ("EP < 2 is local only"): the permute of moe_permute with
 * the rows written straight into the 128-aligned receive layout xr [moe_recv_rows_max, d]
 * (by local slot, padding rows zeroed) and the layout record written -- exactly the xr and
 * layout moe_permute + moe_dispatch produce, without the send-layout copy xs and the
 * transfer.  counts are moe_permute's; dest_row holds each kept slot's row IN xr (the receive
 * layout; -1 = dropped), so the rest of the EP = 1 layer works on the receive layout in place:
 * moe_expert_ffn -> moe_unpermute(out, ...) forward, moe_combine_bwd_local ->
 * moe_expert_ffn_bwd -> moe_permute_bwd(_router)(dxr, ...) backward, with no send-layout
 * buffers and no completion flags.  xr need not be symmetric.  MOE_ERR_INVALID_ARG unless
 * ep_size == 1. */
moe_status moe_permute_dispatch_local(moe_ctx* ctx, const moe_bf16* x, const int32_t* topk_idx,
                                      int32_t* counts, int32_t* dest_row, int32_t* layout,
                                      moe_bf16* xr, moe_stream stream);
/* F6 alone: y[t] = bf16( sum_{j kept} gates[t,j] * rows[dest_row[t,j]] (j order, fp32)
 * + y_extra[t] ), one rounding; y_extra may be NULL.  rows: [*, d] in whatever layout
 * dest_row indexes (the send layout after moe_combine, the receive layout after
 * moe_permute_dispatch_local). */
moe_status moe_unpermute(moe_ctx* ctx, const moe_bf16* rows, const float* gates,
                         const int32_t* dest_row, const moe_bf16* y_extra, moe_bf16* y,
                         moe_stream stream);
/* B6 at EP = 1 on the receive layout (dest_row from moe_permute_dispatch_local): for every kept
 * slot dout_r[dest_row] = bf16(gates * dy[t]) and dgates = <dy[t], out[dest_row]> (fp32, a
 * fixed order -- bit-identical to moe_combine_bwd's), 0 for dropped slots; the padding rows of
 * dout_r's segments (layout record) are zeroed.  out: the expert outputs [recv_rows_max, d]
 * (moe_expert_ffn).  MOE_ERR_INVALID_ARG unless ep_size == 1. */
moe_status moe_combine_bwd_local(moe_ctx* ctx, const moe_bf16* dy, const float* gates,
                                 const int32_t* dest_row, const moe_bf16* out,
                                 const int32_t* layout, float* dgates, moe_bf16* dout_r,
                                 moe_stream stream);
/* dx[t] = bf16( sum_{j kept} dxs[dest_row[t,j]]  (fp32, j order)
 *               + dx_acc[t] (fp32, optional) + dx_extra[t] (bf16, optional) ), one rounding. */
moe_status moe_permute_bwd(moe_ctx* ctx, const moe_bf16* dxs, const int32_t* dest_row,
                           const float* dx_acc_or_null, const moe_bf16* dx_extra_or_null,
                           moe_bf16* dx, moe_stream stream);
/* B2 fused with the dgrad half of B0, for k > 1 (MOE_ERR_INVALID_ARG for k = 1): with the
 * gate a softmax over the k selected logits (reading R1) dlogits[t,:] is zero outside
 * topk_idx[t,:], so dx_router[t] = sum_j dlogits[t,e_j] w_r[e_j,:] is a k-row gather:
 *   dx[t] = bf16( sum_{j kept} dxs[dest_row[t,j]] + sum_j dlogits[t,e_j] w_r[e_j,:]
 *                 + dx_extra[t] (optional) )   in fp32, one rounding.
 * Equivalent to moe_router_logits_bwd(dx_router) + moe_permute_bwd(dx_acc = dx_router)
 * without materialising the fp32 [T_local, d] dx_router. */
moe_status moe_permute_bwd_router(moe_ctx* ctx, const moe_bf16* dxs, const int32_t* dest_row,
                                  const int32_t* topk_idx, const float* dlogits,
                                  const moe_bf16* w_r, const moe_bf16* dx_extra_or_null,
                                  moe_bf16* dx, moe_stream stream);

/* ---------------- F3 / B3 dispatch all-to-all ---------------- */

/* Collective.  Exchanges counts into the [EP x E] matrix, writes the layout record,
 * then stores every send row of xs directly into its owner's xr (NVSwitch peer
 * stores; local rows by plain stores) at the receive layout above, zeroes xr's
 * padding rows, and waits until all peers' rows have landed.  xr: symmetric,
 * moe_recv_rows_max() rows. */
moe_status moe_dispatch(moe_ctx* ctx, const moe_bf16* xs, const int32_t* counts,
                        int32_t* layout, moe_bf16* xr, moe_stream stream);
/* Collective.  Reverse pattern: owner rows of dxr go back to the same send-layout rows
 * of each source's dxs (symmetric, [T_local*k, d]). */
moe_status moe_dispatch_bwd(moe_ctx* ctx, const moe_bf16* dxr, const int32_t* layout,
                            moe_bf16* dxs, moe_stream stream);

/* ---------------- F4 / B4 grouped SwiGLU expert FFN -------- */

/* For each group g (a local expert, or the shared experts as one group of width f):
 *   G = X_g W_gate, U = X_g W_up, H = silu(G)*U, O_g = H W_down   (reading R8)
 * X_g = rows [seg_base[g], seg_base[g]+group_rows[g]) of xr with seg_base the
 * MOE_ALIGN_ROWS-aligned prefix of group_rows (device int32 [n_groups]).  bf16 operands,
 * fp32 accumulation in TMEM (tcgen05), one bf16 rounding per output.
 *   g_u_h [rows_cap, 3f] bf16 saved for backward: cols [0,f)=G, [f,2f)=U, [2f,3f)=H
 *   out   [rows_cap, d]  bf16
 * Padding rows inside a segment are written as zeros; nothing at or beyond rows_cap is
 * written.  f must be a multiple of 128. */
moe_status moe_expert_ffn(moe_ctx* ctx, const moe_bf16* xr, const int32_t* group_rows,
                          int32_t n_groups, int64_t rows_cap, int32_t f,
                          const moe_bf16* w_gu, const moe_bf16* w_down,
                          moe_bf16* g_u_h, moe_bf16* out, moe_stream stream);
/* Backward of moe_expert_ffn given dout [rows_cap, d] (padding rows must be zero):
 *   dH = dout W_down^T; dG = dH*U*silu'(G); dU = dH*silu(G)   -> dgu [rows_cap, 2f] bf16
 *   dxr = dG W_gate^T + dU W_up^T                              -> [rows_cap, d] bf16
 *   dw_down[g] (+)= H^T dout, dw_gu[g] (+)= X^T [dG dU]        -> fp32, same layouts as
 *   the weights; accumulate != 0 adds to the existing values.  dgu is caller scratch. */
moe_status moe_expert_ffn_bwd(moe_ctx* ctx, const moe_bf16* xr, const int32_t* group_rows,
                              int32_t n_groups, int64_t rows_cap, int32_t f,
                              const moe_bf16* w_gu, const moe_bf16* w_down,
                              const moe_bf16* g_u_h, const moe_bf16* dout, moe_bf16* dgu,
                              moe_bf16* dxr, float* dw_gu, float* dw_down, int accumulate,
                              moe_stream stream);

/* ---------------- fused compute + all-to-all (PAPER.md:126 overlap
 * within MoE layers) ---------------- */

/* Collective.  F4 + F5 + F6 in one call for the routed experts of this rank (n_groups = E_l,
 * group rows and receive segments from `layout`, rows_cap = moe_recv_rows_max): GEMM1 +
 * SwiGLU, then GEMM2 whose epilogue stores every output row O[w] of local expert e_l from
 * source r straight into rank r's ys (symmetric) at the send-layout row -- NVSwitch peer
 * stores overlapped with the GEMM's own tiles, no local O buffer and no separate transfer
 * kernel -- then waits for every rank's rows and computes y as moe_combine does.
 * Bit-identical results to moe_expert_ffn + moe_combine. */
moe_status moe_expert_ffn_combine(moe_ctx* ctx, const moe_bf16* xr, const int32_t* layout,
                                  const moe_bf16* w_gu, const moe_bf16* w_down, moe_bf16* g_u_h,
                                  moe_bf16* ys, const float* gates, const int32_t* dest_row,
                                  const moe_bf16* y_extra_or_null, moe_bf16* y, moe_stream stream);
/* Collective.  F3 + F4 (up) in ONE launch, the tile-granular dispatch -> GEMM1 overlap
 * ("computation-communication overlap within MoE layers"; volumes and receive
 * placement PAPER.md:354-356).  Same arguments and results as moe_dispatch(xs, counts,
 * layout, xr) followed by moe_expert_ffn_up(xr, layout, 0, E_l, w_gu, g_u_h) -- xr, the
 * layout record and g_u_h bit-identical -- but inside the persistent GEMM1 launch: two warps
 * of every CTA push this rank's rows to their owners (NVSwitch peer stores) and release a
 * per-(owner slot, source) arrival flag as each segment completes, and every GEMM1 tile
 * starts as soon as the rows of its 128-row A box have arrived instead of after the whole
 * exchange.  xr must be a symmetric allocation of moe_recv_rows_max rows (else
 * MOE_ERR_NOT_SYMMETRIC); f % 128 == 0; counts [E] device int32 from moe_permute; xs may be
 * NULL when T_local == 0.  Follow with moe_expert_ffn_down_combine.  A peer that never
 * arrives faults the kernel after 10 s (MOE_ERR_TIMEOUT in the device error word). */
moe_status moe_dispatch_expert_ffn_up(moe_ctx* ctx, const moe_bf16* xs, const int32_t* counts,
                                      int32_t* layout, moe_bf16* xr, const moe_bf16* w_gu,
                                      moe_bf16* g_u_h, moe_stream stream);
/* Collective.  B6+B5 + B4 (dgrad-1) in ONE launch, the backward twin of
 * moe_dispatch_expert_ffn_up: same arguments and results as moe_combine_bwd(dy, gates,
 * dest_row, ys, layout, dgates, dout_r) followed by moe_expert_ffn_bwd_dh(layout, 0, E_l,
 * w_down, g_u_h, dout_r, dgu) -- dout_r, dgates and dgu bit-identical -- with the transfer
 * run by two warps of every dgrad-1 CTA in slot-major order (row r of the send layout carries
 * bf16(g[t,j] dy[t]) for the slot (t,j) that moe_permute placed there; dgates[t,j] =
 * <dy[t], ys[r]>) and every dO tile started as soon as its rows have arrived.  Requires the
 * moe_permute of the same step (its row -> slot map) and the forward's layout record;
 * dout_r symmetric of moe_recv_rows_max rows; f % 128 == 0.  Follow with
 * moe_expert_ffn_bwd_dx_dispatch. */
moe_status moe_combine_bwd_expert_ffn_dh(moe_ctx* ctx, const moe_bf16* dy, const float* gates,
                                         const int32_t* dest_row, const moe_bf16* ys,
                                         const int32_t* layout, float* dgates, moe_bf16* dout_r,
                                         const moe_bf16* w_down, const moe_bf16* g_u_h,
                                         moe_bf16* dgu, moe_stream stream);
/* Collective.  B4 + B3 in one call: as moe_expert_ffn_bwd for the routed experts, but the
 * dgrad-2 epilogue stores every dX row straight into its source rank's dxs (symmetric) at
 * the send-layout row; the weight-gradient GEMMs run while those stores drain, and the call
 * ends by waiting for every rank's rows.  Bit-identical to moe_expert_ffn_bwd +
 * moe_dispatch_bwd. */
moe_status moe_expert_ffn_bwd_dispatch(moe_ctx* ctx, const moe_bf16* xr, const int32_t* layout,
                                       const moe_bf16* w_gu, const moe_bf16* w_down,
                                       const moe_bf16* g_u_h, const moe_bf16* dout, moe_bf16* dgu,
                                       moe_bf16* dxs, float* dw_gu, float* dw_down, int accumulate,
                                       moe_stream stream);

/* ---------------- chunked overlap of the all-to-alls with the expert GEMMs (NEXT-1:
 * "chunked dispatch -> GEMM") ----------------
 * The owner slots [0, E_l) are cut into ranges.  The transfer of range c+1 runs on a second
 * stream (moe_ctx_set_sm_limits gives it comm_sms SMs) while the first expert GEMM of range c
 * runs on this one; no kernel ever waits for a kernel of the other stream, so the two
 * launches cannot deadlock whatever the SM scheduler does.  Every range call is a
 * collective (all ranks, same ranges, same order).  Results are bit-identical to the
 * unchunked calls: the ranges partition the rows, and every output row is computed by the
 * same kernel code with the same operands.
 *
 *   forward : moe_dispatch_range(r0) ; [moe_dispatch_range(r1) || moe_expert_ffn_up(r0)] ;
 *             ... ; moe_expert_ffn_up(r_last) ; moe_expert_ffn_down_combine
 *   backward: moe_combine_bwd_range(r0) ; [moe_combine_bwd_range(r1) || moe_expert_ffn_bwd_dh(r0)] ;
 *             ... ; moe_expert_ffn_bwd_dh(r_last) ; moe_expert_ffn_bwd_dx_dispatch
 */

/* Collective.  moe_dispatch for the rows bound to owner slots [slot_begin, slot_end) only
 * (padding rows of those slots zeroed).  The range with slot_begin == 0 must come first in
 * a step: it exchanges the counts and writes the whole layout record; the later ranges read
 * the counts from that record (counts may then be NULL).  moe_dispatch == the range
 * [0, E_l).  0 <= slot_begin < slot_end <= E_l, else MOE_ERR_INVALID_ARG. */
moe_status moe_dispatch_range(moe_ctx* ctx, const moe_bf16* xs, const int32_t* counts_or_null,
                              int32_t* layout, moe_bf16* xr, int32_t slot_begin,
                              int32_t slot_end, moe_stream stream);
/* Collective.  moe_combine_bwd for the rows bound to owner slots [slot_begin, slot_end):
 * their dO rows and dgates entries (dropped slots' dgates = 0 are written by the range with
 * slot_begin == 0).  moe_combine_bwd == the range [0, E_l). */
moe_status moe_combine_bwd_range(moe_ctx* ctx, const moe_bf16* dy, const float* gates,
                                 const int32_t* dest_row, const moe_bf16* ys,
                                 const int32_t* layout, float* dgates, moe_bf16* dout_r,
                                 int32_t slot_begin, int32_t slot_end, moe_stream stream);
/* Not collective.  GEMM1 + SwiGLU (G, U, H into g_u_h) for the local experts in slots
 * [slot_begin, slot_end), rows from the layout record. */
moe_status moe_expert_ffn_up(moe_ctx* ctx, const moe_bf16* xr, const int32_t* layout,
                             int32_t slot_begin, int32_t slot_end, const moe_bf16* w_gu,
                             moe_bf16* g_u_h, moe_stream stream);
/* Collective.  The rest of moe_expert_ffn_combine after every range's moe_expert_ffn_up:
 * GEMM2 with the combine stores fused into its epilogue, the flag wait and y. */
moe_status moe_expert_ffn_down_combine(moe_ctx* ctx, const int32_t* layout,
                                       const moe_bf16* w_down, moe_bf16* g_u_h, moe_bf16* ys,
                                       const float* gates, const int32_t* dest_row,
                                       const moe_bf16* y_extra_or_null, moe_bf16* y,
                                       moe_stream stream);
/* Not collective.  dgrad-1 + dSwiGLU (dG, dU into dgu) for slots [slot_begin, slot_end). */
moe_status moe_expert_ffn_bwd_dh(moe_ctx* ctx, const int32_t* layout, int32_t slot_begin,
                                 int32_t slot_end, const moe_bf16* w_down, const moe_bf16* g_u_h,
                                 const moe_bf16* dout, moe_bf16* dgu, moe_stream stream);
/* Collective.  The rest of moe_expert_ffn_bwd_dispatch after every range's
 * moe_expert_ffn_bwd_dh: dgrad-2 with the dispatch_bwd stores fused, both weight-gradient
 * GEMMs, the flag wait. */
moe_status moe_expert_ffn_bwd_dx_dispatch(moe_ctx* ctx, const moe_bf16* xr, const int32_t* layout,
                                          const moe_bf16* w_gu, const moe_bf16* g_u_h,
                                          const moe_bf16* dout, const moe_bf16* dgu, moe_bf16* dxs,
                                          float* dw_gu, float* dw_down, int accumulate,
                                          moe_stream stream);

/* ---------------- F5+F6 / B6+B5 combine ("same communication in the
 * reverse direction") ---------------- */

/* Collective.  Owner rows of `out` go back to the same send-layout rows of each
 * source's ys (symmetric [T_local*k, d]); then
 *   y[t] = bf16( sum_{j kept} gates[t,j] * ys[dest_row[t,j]] (fp32, j order)
 *                + y_extra[t] (bf16 shared-expert output, optional) ). */
moe_status moe_combine(moe_ctx* ctx, const moe_bf16* out, const int32_t* layout,
                       moe_bf16* ys, const float* gates, const int32_t* dest_row,
                       const moe_bf16* y_extra_or_null, moe_bf16* y, moe_stream stream);
/* Collective.  dgates[t,j] = <dy[t], ys[dest_row[t,j]]> (fp32; 0 for dropped slots);
 * dO rows g[t,j]*dy[t] (bf16) are stored straight into their owner's dout_r
 * (symmetric, moe_recv_rows_max() rows; padding rows zeroed) at the receive layout. */
moe_status moe_combine_bwd(moe_ctx* ctx, const moe_bf16* dy, const float* gates,
                           const int32_t* dest_row, const moe_bf16* ys, const int32_t* layout,
                           float* dgates, moe_bf16* dout_r, moe_stream stream);

/* ---------------- NEXT-4 deduplicated all-to-all (reading R18) -------
 * The plain dispatch sends one row per kept slot (t, j); a token whose k experts share an
 * owner crosses NVLink several times with the same bytes.  Here a token crosses once per
 * (token, owner) PAIR -- X-MoE's "redundancy-based communication bypassing",
 * the single-box form of the paper's hierarchical all-to-all (which reduces
 * to its Phase I inside one switch group).  oracle/dedup.py is the definition:
 *   pair (t, q)  iff some kept slot j of token t has owner(e_j) = q; tslot = rank of t among
 *                this rank's tokens paired with q (ascending t); ntok[q] = pairs with q.
 *   source pair rows   pdest[t, q] = pair_base[q] + tslot  (pair_base = exclusive scan of
 *                      ntok over q), -1 if no pair; rows of part / dxpart / dgpart.
 *   owner token rows   u = tok_base[r] + tslot for pairs from source r, tok_base[r] =
 *                      sum_{r'<r} ntok_all[r'][me]; rows of xt / dyt, rlist, glist, dg_own.
 *   rlist[u][j]        receive row (the plain receive layout above) of slot j of the pair's
 *                      token if kept and owned here, else -1; glist[u][j] its gate (else 0).
 *   pair record        dlayout [EP*EP] int32 = ntok_all[r][q], written by moe_dedup_dispatch.
 * Every other tensor (xr, out, dout_r, dxr, the layout record) is exactly the plain path's, so
 * the expert FFN calls are unchanged.  The combine partials are rounded to bf16 once on the
 * owner, so y and dx carry a second bf16 rounding (inside the 2e-2 tolerance, reading R18).
 * Symmetric buffers (moe_symm_alloc): xt/dyt [moe_dedup_token_rows_max, d] bf16, rlist, glist
 * [moe_dedup_token_rows_max, k] (owner side); part, dxpart [moe_dedup_pair_rows_max, d] bf16,
 * dgpart [moe_dedup_pair_rows_max, k] fp32 (source side). */

/* T_local * min(k, EP): bound on a source's pair rows; -1 for an invalid shape. */
int64_t moe_dedup_pair_rows_max(const moe_shape* shape);
/* min(EP * T_local, moe_recv_rows_max): bound on an owner's token rows; -1 if invalid. */
int64_t moe_dedup_token_rows_max(const moe_shape* shape);

/* Not collective.  pdest [T_local, EP] int32 and ntok [EP] int32 from topk_idx and
 * dest_row (moe_permute's output; xs may be NULL there) under the ctx's expert placement. */
moe_status moe_dedup_pairs(moe_ctx* ctx, const int32_t* topk_idx, const int32_t* dest_row,
                           int32_t* pdest, int32_t* ntok, moe_stream stream);
/* Collective.  F3 deduplicated: exchanges counts and ntok, writes the layout record (as
 * moe_dispatch) and the pair record dlayout, stores each paired x row once into its owner's
 * xt (each 2 KB part of x[t] is read once and stored to every owner of t) with the pair's
 * rlist / glist rows, waits for every peer, then expands locally: xr[rlist[u][j]] = xt[u],
 * padding rows zeroed.  xr is bit-identical to moe_dispatch's (it need not be symmetric). */
moe_status moe_dedup_dispatch(moe_ctx* ctx, const moe_bf16* x, const int32_t* counts,
                              const int32_t* ntok, const int32_t* pdest, const int32_t* dest_row,
                              const int32_t* topk_idx, const float* gates, int32_t* layout,
                              int32_t* dlayout, moe_bf16* xt, int32_t* rlist, float* glist,
                              moe_bf16* xr, moe_stream stream);
/* Collective.  F5+F6 deduplicated: per pair the owner forms
 *   part[u] = bf16( sum_{j: rlist[u][j] >= 0} glist[u][j] * out[rlist[u][j]] )  (fp32, j order)
 * and stores it at the source's pair row; after every peer's rows arrived
 *   y[t] = bf16( sum_q part[pdest[t,q]] (fp32, q ascending) + y_extra[t] (optional) ). */
moe_status moe_dedup_combine(moe_ctx* ctx, const moe_bf16* out, const int32_t* dlayout,
                             const int32_t* rlist, const float* glist, const int32_t* pdest,
                             const moe_bf16* y_extra_or_null, moe_bf16* part, moe_bf16* y,
                             moe_stream stream);
/* Collective.  B6+B5 deduplicated: dy[t] crosses once per pair into the owner's dyt; then,
 * locally on the owner, dout_r[rl] = bf16(g * dyt[u]) and dg_own[u][j] = <dyt[u], out[rl]>
 * (fp32; 0 where rlist < 0) -- O never leaves its owner.  dout_r padding rows zeroed. */
moe_status moe_dedup_combine_bwd(moe_ctx* ctx, const moe_bf16* dy, const int32_t* pdest,
                                 const int32_t* layout, const int32_t* dlayout,
                                 const int32_t* rlist, const float* glist, const moe_bf16* out,
                                 moe_bf16* dyt, float* dg_own, moe_bf16* dout_r,
                                 moe_stream stream);
/* Collective.  B6+B5 with the dispatch direction deduplicated and the combine left to the
 * fused GEMM2 stores (moe_expert_ffn_combine: O rows already sit in this rank's ys):
 *   dgates[t,j] = <dy[t], ys[dest_row[t,j]]> (fp32, 0 for dropped slots) at the source, dy[t]
 * once per pair into the owner's dyt, then on the owner dout_r[rl] = bf16(g * dyt[u]) (padding
 * rows zeroed).  Bit-identical dgates and dout_r to moe_combine_bwd. */
moe_status moe_dedup_combine_bwd_ys(moe_ctx* ctx, const moe_bf16* dy, const float* gates,
                                    const int32_t* dest_row, const moe_bf16* ys,
                                    const int32_t* pdest, const int32_t* layout,
                                    const int32_t* dlayout, const int32_t* rlist,
                                    const float* glist, moe_bf16* dyt, float* dgates,
                                    moe_bf16* dout_r, moe_stream stream);
/* Collective.  B3 deduplicated: dxpart[pair row] = bf16( sum_j dxr[rlist[u][j]] ) (fp32, j
 * order) and dgpart[pair row][j] = dg_own[u][j] go to each source; then locally
 * dgates[t,j] = dgpart[pdest[t, owner(e_j)]][j] (0 for dropped slots). */
moe_status moe_dedup_dispatch_bwd(moe_ctx* ctx, const moe_bf16* dxr, const int32_t* dlayout,
                                  const int32_t* rlist, const float* dg_own, const int32_t* pdest,
                                  const int32_t* dest_row, const int32_t* topk_idx,
                                  moe_bf16* dxpart, float* dgpart, float* dgates,
                                  moe_stream stream);
/* B2 + B0 dgrad as moe_permute_bwd_router (k > 1), rows from the pair buffer:
 *   dx[t] = bf16( sum_q dxpart[pdest[t,q]] + sum_j dlogits[t,e_j] w_r[e_j,:] + dx_extra[t] ). */
moe_status moe_dedup_permute_bwd_router(moe_ctx* ctx, const moe_bf16* dxpart,
                                        const int32_t* pdest, const int32_t* topk_idx,
                                        const float* dlogits, const moe_bf16* w_r,
                                        const moe_bf16* dx_extra_or_null, moe_bf16* dx,
                                        moe_stream stream);

/* ---------------- NEXT-3 PP x EP pipelined executor ----------------
 * P GPUs as a PP x EP mesh -- PP pipeline stages, each staffed by EP GPUs holding
 * L/PP MoE layers with E/EP experts per GPU; the 1F1B schedule keeps at
 * most PP - i micro-batches in flight on stage i.  The layer calls above are unchanged; the
 * executor (paper_2605_05049_b200/pipeline.py) runs this op list per stage. */
#define MOE_PIPE_FORWARD 0
#define MOE_PIPE_BACKWARD 1
/* Host function (no GPU).  The op list of `stage` (reading R19): ops[2i] = MOE_PIPE_FORWARD or
 * MOE_PIPE_BACKWARD, ops[2i+1] = micro-batch; *n_ops = 2 * n_micro.  MOE_ERR_INVALID_ARG for
 * pp < 1, stage outside [0, pp), n_micro < 1, max_ops < 2 * n_micro or NULL pointers. */
moe_status moe_pipeline_1f1b(int32_t pp, int32_t stage, int32_t n_micro, int32_t* ops,
                             int32_t max_ops, int32_t* n_ops);

#ifdef __cplusplus
}
#endif
#endif /* MOE_H_ */
