// internal.h -- host-side interfaces between the C-ABI layer (api.cu) and the
// kernel translation units.  Not installed; not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "../../include/moe.h"

namespace moe {

// ---------------------------------------------------------------- launches
// Programmatic dependent launch for every libmoe kernel (common.cuh pdl_wait / pdl_trigger)
// unless MOE_PDL=0.
inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}
inline int pdl_attr(cudaLaunchAttribute* attr) {
  if (!pdl_enabled()) return 0;
  attr->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  cfg.numAttrs = pdl_attr(attr);
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- grouped GEMM
// One persistent tcgen05 kernel family serves every dense contraction of the
// layer: D[M,N] = A[M,K] * B[N,K]^T per group.
enum Epilogue : int {
  kEpiSwiGLU = 0,   // GEMM1 fwd: acc cols [0,BN/2)=G, [BN/2,BN)=U -> G,U,H bf16 into g_u_h
  kEpiBF16 = 1,     // plain bf16 store (GEMM2 fwd O, dgrad dX)
  kEpiDSwiGLU = 2,  // dgrad-1: acc = dH; reads G,U -> dG,dU bf16 into dgu
  kEpiF32Group = 3, // wgrad: fp32 [M,N] per group (K = the group's rows), optional accumulate
  kEpiF32Rows = 4,  // router logits: fp32 [rows,N] + bias
  kEpiSwiGLUDisp = 5,  // GEMM1 + SwiGLU with the dispatch all-to-all fused in (NEXT-1):
                       // warps 2-3 push this rank's send rows to their owners while the
                       // producer starts each A tile as soon as its source rows have landed
  kEpiDSwiGLUComb = 6, // dgrad-1 + dSwiGLU with combine_bwd fused in (NEXT-1, backward twin):
                       // warps 2-3 push g * dy rows (and compute dgates), each dO tile starts
                       // when its rows have landed
};

struct GemmProblem {
  int epi = kEpiBF16;
  int BN = 256;
  bool a_mn = false, b_mn = false;  // operand major-ness in global memory (MN = contiguous along M/N)
  // A / B global tensors (bf16, row-major [rows, cols] with leading dimension ld elements)
  const void* a_ptr = nullptr;
  int64_t a_rows = 0, a_cols = 0, a_ld = 0;
  const void* b_ptr = nullptr;
  int64_t b_rows = 0, b_cols = 0, b_ld = 0;
  int64_t b_group_stride = 0;  // rows of B per group when B holds weights
  int64_t b_split = 0;         // SwiGLU: row offset of W_up inside a group (= f)
  int M = 0, N = 0, K = 0;     // M-grouped: N, K; K-grouped: M, N
  const int32_t* group_rows = nullptr;  // device [n_groups]
  int n_groups = 0;
  int group_begin = 0;  // M-grouped: tiles only for groups [group_begin, n_groups)
  int64_t rows_cap = 0;
  void* out = nullptr;
  int64_t ld_out = 0;
  const void* aux = nullptr;  // DSwiGLU: g_u_h
  int64_t ld_aux = 0;
  const float* bias = nullptr;
  int f = 0;
  int accumulate = 0;
  int n_fastest = 0;  // tile raster order: 1 = n fastest (re-read B), 0 = m fastest (re-read A)
  int max_ctas = 0;   // SM budget (0 = all SMs); used to run a GEMM beside a transfer
  int pair = 1;       // 2: CTA-pair tiles (tcgen05 cta_group::2, M = 256), BN >= 128 only
  // kEpiBF16 only: fused reverse all-to-all (rows -> source ranks' symmetric buffer at
  // scatter_off), the kernel's last CTA publishes comm->epoch on the data flags
  int scatter = 0;
  int64_t scatter_off = 0;
  const int32_t* scatter_layout = nullptr;  // counts_all [EP x E]
  const struct CommArgs* comm = nullptr;
  // kEpiSwiGLUDisp only (group_rows unused: the group tables come from the counts exchange)
  const void* disp_src = nullptr;      // send layout xs [T*k, d] (this rank's rows)
  const int32_t* disp_counts = nullptr;  // this rank's per-expert counts [E]
  int32_t* disp_layout = nullptr;      // layout record written by the kernel
  int64_t disp_dst_off = 0;            // byte offset of xr (= a_ptr) inside every heap
  int64_t arrive_off = 0;              // heap offset of the arrival flags [E_l][EP+1]
  int32_t* disp_work = nullptr;        // local scratch, zero between calls: [4 + E + E_l]
  // kEpiDSwiGLUComb: combine_bwd payload sources (disp_dst_off = dout_r, arrive/work as above)
  const void* cb_dy = nullptr;            // dy [T_local, d]
  const float* cb_gates = nullptr;        // [T_local * k]
  const void* cb_ys = nullptr;            // ys [T_local * k, d] (send layout, forward outputs)
  float* cb_dgates = nullptr;             // [T_local * k] out
  const int32_t* cb_slot_of_row = nullptr;  // send-layout row -> slot t*k+j
  const int32_t* cb_dest_row = nullptr;   // [T_local * k] (-1: dropped -> dgates 0)
  const int32_t* cb_layout = nullptr;     // layout record of the forward dispatch
};

cudaError_t launch_grouped_gemm(const GemmProblem& p, cudaStream_t stream);
int num_sms();

// ---------------------------------------------------------------- routing / permutation
cudaError_t launch_route(const float* logits, int64_t T, int E, int k, int32_t* topk_idx,
                         float* gates, cudaStream_t s);
cudaError_t launch_route_bwd(const float* logits, const int32_t* topk_idx, const float* gates,
                             const float* dgates, int64_t T, int E, int k, float* dlogits,
                             cudaStream_t s);
cudaError_t launch_split_hilo(const float* dl, int64_t T, int E, int Ep, uint16_t* out,
                              cudaStream_t s);
cudaError_t launch_stack_wr(const uint16_t* w_r, int E, int Ep, int d, uint16_t* out,
                            cudaStream_t s);
cudaError_t launch_permute_bwd_router(const uint16_t* dxs, const int32_t* dest_row,
                                      const int32_t* topk_idx, const float* dlogits,
                                      const uint16_t* w_r, const uint16_t* dx_extra, int64_t T,
                                      int d, int E, int k, uint16_t* dx, cudaStream_t s);
cudaError_t launch_sum_partials(const float* part, int S, int E, int Ep, int d, float* dw,
                                int accumulate, cudaStream_t s);
// scratch: int32 workspace of permute_scratch_ints(T,k,E) entries
int64_t permute_scratch_ints(int64_t T, int k, int E);
// layout != null: EP = 1 local path -- xs is then the 128-aligned receive buffer (rows placed
// by slot, expert_at[slot] = expert, padding zeroed; pad_rows_max bounds the padding rows) and
// the layout record is written, as moe_dispatch would
cudaError_t launch_permute(const uint16_t* x, const int32_t* topk_idx, int64_t T, int d, int E,
                           int k, int64_t C, int32_t* counts, int32_t* dest_row, uint16_t* xs,
                           int32_t* scratch, cudaStream_t s, int32_t* layout = nullptr,
                           const int32_t* expert_at = nullptr, int64_t pad_rows_max = 0,
                           int32_t* slot_of_row = nullptr);
cudaError_t launch_permute_bwd(const uint16_t* dxs, const int32_t* dest_row, const float* dx_acc,
                               const uint16_t* dx_extra, int64_t T, int d, int k, uint16_t* dx,
                               cudaStream_t s);
// B2 + B0 dgrad with a row-list width kr independent of k (dedup pair rows: kr = EP)
cudaError_t launch_permute_bwd_router_rows(const uint16_t* dxs, const int32_t* rows, int kr,
                                           const int32_t* topk_idx, const float* dlogits,
                                           const uint16_t* w_r, const uint16_t* dx_extra,
                                           int64_t T, int d, int E, int k, uint16_t* dx,
                                           cudaStream_t s);
// NEXT-4 dedup, source side (reading R18): pdest [T,EP] = pair row of (t, q) or -1,
// ntok [EP] pairs per owner; one block
// scratch: int32 workspace of dedup_scratch_ints(T, EP) entries, zeroed once (ticket)
int64_t dedup_scratch_ints(int64_t T, int EP);
cudaError_t launch_dedup_pairs(const int32_t* topk_idx, const int32_t* dest_row,
                               const int32_t* place, int64_t T, int k, int E_l, int EP,
                               int32_t* pdest, int32_t* ntok, int32_t* scratch, cudaStream_t s);
// dgates[t,j] = dgpart[pdest[t, owner(e_j)] * k + j] (0 for dropped slots)
cudaError_t launch_dedup_dgates(const int32_t* dest_row, const int32_t* topk_idx,
                                const int32_t* pdest, const int32_t* place, int E_l, int EP,
                                const float* dgpart, int64_t T, int k, float* dgates,
                                cudaStream_t s);
// B6 at EP = 1 on the receive layout (dest_row = receive rows): dout rows = g * dy, dgates =
// <dy, O rows>; zeroes the padding rows of dout's segments (layout record)
cudaError_t launch_combine_bwd_local(const uint16_t* dy, const float* gates,
                                     const int32_t* dest_row, const uint16_t* O,
                                     const int32_t* layout, int64_t T, int d, int k, int E,
                                     int64_t pad_rows_max, float* dgates, uint16_t* dout,
                                     cudaStream_t s);
cudaError_t launch_unpermute(const uint16_t* ys, const float* gates, const int32_t* dest_row,
                             const uint16_t* y_extra, int64_t T, int d, int k, uint16_t* y,
                             cudaStream_t s);

// ---------------------------------------------------------------- transfers (NVSwitch)
struct PeerTable {
  char* base[MOE_MAX_EP];  // symmetric heap base of every rank, mapped into this process
};

struct CommArgs {
  PeerTable peers;
  int ep, rank, E, E_l, d;
  int64_t T, k;
  uint64_t* flags;       // local flag array [n_slots][EP] in the symmetric heap
  int64_t flags_off;     // byte offset of the flag array inside every heap
  int32_t* countmat;     // local count matrix [2][EP][E] in the symmetric heap
  int64_t countmat_off;
  int32_t* ntokmat;      // local pair-count matrix [2][EP][EP] (dedup all-to-all, NEXT-4)
  int64_t ntokmat_off;
  int32_t* done;         // local device counter for last-block detection
  int32_t* err;          // device error word
  // Per-call epoch (identical on every rank): kernels read *epoch_ptr + 1 at their start and
  // the LAST kernel of a collective stores it back once every peer's flag has arrived, so the
  // counter lives on the device and the whole step can be replayed from a CUDA graph.
  uint64_t* epoch_ptr;
  uint64_t epoch;        // set on the device at kernel start (load_epoch)
  int blocks;            // transfer kernel blocks (0 = 2 per SM)
  // expert placement (NEXT-2 migration): place[e] = global slot of expert e (owner =
  // slot / E_l, local slot = slot % E_l), expert_at = its inverse; device [E] each
  const int32_t* place;
  const int32_t* expert_at;
};
enum { kSlotCounts = 0, kSlotData = 1, kNumSlots = 2 };

// Heap base of rank q: a select chain over static indices, so the kernel-parameter copy of the
// peer table is never indexed dynamically (that forced a 208-byte local-memory frame).
#ifdef __CUDACC__
__device__ __forceinline__ char* peer_base(const CommArgs& a, int q) {
  char* p = a.peers.base[0];
#pragma unroll
  for (int i = 1; i < MOE_MAX_EP; ++i)
    if (q == i) p = a.peers.base[i];
  return p;
}
#endif

// Each collective is ONE launch that returns only when this rank's destination buffer is
// complete (the last block waits for every peer's flag).  dst_off = byte offset of the
// destination buffer inside every rank's symmetric heap.
// Forward pattern (source send-layout rows -> owners' receive rows; zeroes local padding):
//   dispatch: counts exchange + layout record + rows of src
// Both move only the rows bound for owner slots [s0, s1) (NEXT-1 chunked overlap); the
// range with s0 == 0 of a dispatch also exchanges the counts and writes the layout record.
cudaError_t launch_dispatch(const CommArgs& a, const int32_t* counts, int32_t* layout,
                            int64_t recv_rows_cap, const uint16_t* src, int64_t dst_off,
                            uint16_t* local_dst, int s0, int s1, cudaStream_t s);
//   combine_bwd: payload rows gates * dy, and dgates = <dy, ys rows>
cudaError_t launch_combine_bwd_transfer(const CommArgs& a, int32_t* layout, int64_t dst_off,
                                        uint16_t* local_dst, const int32_t* dest_row,
                                        const float* gates, const uint16_t* dy, const uint16_t* ys,
                                        float* dgates, int s0, int s1, cudaStream_t s);
// Reverse pattern: owner receive rows -> sources' send-layout rows
cudaError_t launch_reverse_transfer(const CommArgs& a, const int32_t* layout, const uint16_t* src,
                                    int64_t dst_off, cudaStream_t s);
// NEXT-4 deduplicated all-to-all (reading R18; oracle/dedup.py).  Token rows cross once per
// (token, owner) pair into the owner's token buffer (tok_off); rlist/glist (rlist_off,
// glist_off: [pair, k]) name each pair's receive rows and gates on the owner.
//   mode 0 (dispatch): counts + pair counts exchange, layout + pair record, x rows, lists
//   mode 1 (combine_bwd): dy rows (pair layout from dlayout); with ys also
//     dgates[t,j] = <dy[t], ys[dest_row[t,j]]> at the source
cudaError_t launch_dedup_forward(const CommArgs& a, int mode, int32_t* layout, int32_t* dlayout,
                                 const int32_t* counts, const int32_t* ntok,
                                 int64_t recv_rows_cap, const uint16_t* src,
                                 const int32_t* pdest, const int32_t* dest_row,
                                 const int32_t* topk_idx, const float* gates, int64_t tok_off,
                                 int64_t rlist_off, int64_t glist_off, const uint16_t* ys,
                                 float* dgates, cudaStream_t s);
// Owner, local: mode 0 xr[rlist[u][j]] = tok[u]; mode 1 dst[rl] = bf16(g * tok[u]) and, with
// O, dg_own[u][j] = <tok[u], O[rl]>; both zero dst's padding rows
cudaError_t launch_dedup_expand(const CommArgs& a, int mode, const int32_t* layout,
                                const int32_t* dlayout, const uint16_t* tok,
                                const int32_t* rlist, const float* glist, const uint16_t* O,
                                uint16_t* dst, float* dg_own, cudaStream_t s);
// Collective, owner -> sources: part[u] = sum_j w_j rows[rlist[u][j]] (mode 0: w = glist;
// mode 1: w = 1, and dg_own[u][*] goes along to dgpart) at the source's pair row
cudaError_t launch_dedup_reduce(const CommArgs& a, int mode, const int32_t* dlayout,
                                const int32_t* rlist, const float* glist, const uint16_t* rows,
                                const float* dg_own, int64_t part_off, int64_t dgpart_off,
                                cudaStream_t s);
// equal-split all-to-all: chunk q of send -> chunk rank of rank q's buffer at dst_off
cudaError_t launch_all_to_all(const CommArgs& a, const void* send, int64_t dst_off,
                              int64_t chunk_bytes, cudaStream_t s);
// NEXT-2 expert migration: moves of this rank's experts (old local slot -> new owner rank
// and local slot); collective, see migrate_kernel
struct MigrateList {
  int n;
  int16_t src_slot[256];
  int16_t dst_rank[256];
  int16_t dst_slot[256];
};
cudaError_t launch_migrate(const CommArgs& a, const MigrateList& ml, const void* src,
                           int64_t dst_off, int64_t bytes_per_expert, cudaStream_t s);
// 1-block wait for every rank's flag of a.epoch (after a GEMM with a fused scatter epilogue)
cudaError_t launch_wait_flags(const CommArgs& a, int slot, cudaStream_t s);

}  // namespace moe
