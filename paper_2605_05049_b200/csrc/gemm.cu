// gemm.cu -- persistent grouped GEMM on the 5th-generation tensor cores (sm_100a).
//
// Serves every dense contraction on the hot path:
//   F0 router logits   x[T,d] . w_r[E,d]^T                           (M-grouped, 1 group)
//   F4 GEMM1           xr_g . w_gu_g^T  -> G,U,H (SwiGLU epilogue)   (M-grouped)
//   F4 GEMM2           H_g  . w_down_g^T -> O                        (M-grouped)
//   B4 dgrad-1         dO_g . w_down_g   -> dH -> dG,dU (dSwiGLU)    (M-grouped, B MN-major)
//   B4 dgrad-2         dGU_g . w_gu_g    -> dX                       (M-grouped, B MN-major)
//   B4 wgrad           dO_g^T H_g, dGU_g^T X_g  (K = the group's rows) (K-grouped, A,B MN-major)
//   B0 router bwd      dl.W_r, dl^T x  (dl as bf16 hi+lo)
// The paper's expert GEMMs are "tall-and-skinny" per expert;
// here all experts of a rank are ONE persistent launch over a (group, m, n) tile list
// built on the device from the routed row counts, so no host round trip is needed.
//
// Structure (one CTA per SM, 256 threads):
//   warp 0      TMA producer   (cp.async.bulk.tensor, 128B swizzle, mbarrier ring)
//   warp 1      MMA issuer     (tcgen05.mma kind::f16, M=128 x N=BN x K=16, fp32 in TMEM)
//   warp 2      TMEM allocator (2 accumulator stages -> epilogue overlaps the next tile)
//   warp 3      group tables (device-side prefix sums of the routed rows)
//   warps 4..7  epilogue       (tcgen05.ld 32x32b -> fused activation -> 128B-swizzled smem
//                               staging -> TMA store / TMA reduce-add, one 4 KB box per warp)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace moe {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes = one 128B-swizzle atom row
constexpr int kThreads = 256;
constexpr int kMaxGroups = 256;
constexpr int kStageBox = 4096;  // per-epilogue-warp staging: 32 rows x 128 bytes
constexpr int kMaxDevices = 64;

struct KParams {
  int M, N, K;
  int n_groups;
  int group_begin;      // tiles only for groups >= group_begin (segment bases still from 0)
  const int32_t* group_rows;
  int64_t rows_cap;
  int64_t b_group_stride, b_split;
  int n_fastest;        // tile raster: 1 = n fastest (B slab re-read), 0 = m fastest
  int direct_store;     // F32Rows only: output pitch not 16B-aligned -> plain stores
  void* out;
  int64_t ld_out;
  const void* aux;
  int64_t ld_aux;
  const float* bias;
  int f;
  int accumulate;
  int aux_tma;          // dSwiGLU: G / U boxes by TMA (tmX) instead of per-lane loads
  // BF16 epilogue fused with the reverse all-to-all (combine / dispatch_bwd): row w of local
  // expert e_l from source r is stored straight into rank r's symmetric buffer at
  // scatter_off, send-layout row soff[r][e_l] + (w - pre[r][e_l]); the last CTA publishes
  // the epoch flag to every rank.  comm.layout = counts_all [EP x E].
  int scatter;
  int64_t scatter_off;
  const int32_t* scatter_layout;
  CommArgs comm;
  // kEpiSwiGLUDisp (NEXT-1): the dispatch fused in front of GEMM1 (see disp_prologue)
  const uint16_t* disp_src;
  const int32_t* disp_counts;
  int32_t* disp_layout;
  int64_t disp_dst_off;
  int64_t arrive_off;
  int32_t* work;
  // kEpiDSwiGLUComb
  const uint16_t* cb_dy;
  const float* cb_gates;
  const uint16_t* cb_ys;
  float* cb_dgates;
  const int32_t* cb_slot_of_row;
  const int32_t* cb_dest_row;
  const int32_t* cb_layout;
};

// STG = staging boxes per epilogue warp.  2 double-buffers the fp32 wgrad epilogue (its K is
// one expert's rows, so a tile's MMAs are short), at the price of one ring stage.  Measured
// on the V3-like rank slice (ncu, profiles/r01/README.md): wgrad 1.63 -> 1.70 ms and
// 3.29 -> 3.41 ms, i.e. slower -- the ring stage is worth more; kept at 1.
constexpr int kWgradStaging = 1;
template <int BN, int PAIR, int STG = 1, int EXTRA = 0>
struct Cfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = (BN / PAIR) * kBK * 2;  // a CTA pair splits B along N
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (196 * 1024 - (STG - 1) * 4 * kStageBox) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int RING = STAGES * STAGE_BYTES;
  static constexpr int ACC_STRIDE = BN < 32 ? 32 : BN;
  static constexpr int TMEM_COLS = (2 * ACC_STRIDE <= 32)    ? 32
                                   : (2 * ACC_STRIDE <= 64)  ? 64
                                   : (2 * ACC_STRIDE <= 128) ? 128
                                   : (2 * ACC_STRIDE <= 256) ? 256
                                                             : 512;
  // ring + epilogue staging + barriers/tables (incl. scatter tables) + alignment slack
  static constexpr int SMEM = RING + 4 * STG * kStageBox + 6144 + 1024 + EXTRA;
};
template <int EPI>
__host__ __device__ constexpr int staging_boxes() { return EPI == kEpiF32Group ? kWgradStaging : 1; }
// fused dispatch tables (6 E + E_l + 3 ints, E <= 256) beyond the common table area
constexpr int kDispSmem = 8192;
template <int EPI>
__host__ __device__ constexpr int extra_smem() {
  return (EPI == kEpiSwiGLUDisp || EPI == kEpiDSwiGLUComb) ? kDispSmem : 0;
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Decoded work tile.
struct Tile {
  int g, m, n, nkb;
  int rows_g;   // valid rows of the group
  int seg;      // first row of the group's segment
};

template <bool KGROUPED, int BN, int TILE_M>
__device__ __forceinline__ Tile decode_tile(int t, const int* s_tile_prefix, const int* s_seg,
                                            const int* s_rows, int n_groups, const KParams& p) {
  int lo = 0, hi = n_groups;  // g with prefix[g] <= t < prefix[g+1]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (s_tile_prefix[mid] <= t) lo = mid; else hi = mid;
  }
  Tile tl;
  tl.g = lo;
  tl.rows_g = s_rows[lo];
  tl.seg = s_seg[lo];
  const int local = t - s_tile_prefix[lo];
  const int mt = KGROUPED ? ceil_div(p.M, TILE_M) : ceil_div(tl.rows_g, TILE_M);
  if (p.n_fastest) {
    const int nt = ceil_div(p.N, BN);
    tl.n = local % nt;
    tl.m = local / nt;
  } else {
    tl.m = local % mt;
    tl.n = local / mt;
  }
  tl.nkb = KGROUPED ? ceil_div(tl.rows_g, kBK) : p.K / kBK;
  return tl;
}

// One thread's 128-byte row of a 32-row box, written 128B-swizzled (16B chunk j of row r at
// chunk j ^ (r & 7)): conflict-free per quarter warp and the layout TMA SWIZZLE_128B expects.
__device__ __forceinline__ void stage_row(uint32_t row_addr, int lane, const uint32_t (&w)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                 w[4 * j + 3]);
}

// Before overwriting the warp's staging box: the previous TMA store must have read it.
__device__ __forceinline__ void staging_acquire(int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}
// After staging: make the writes visible to the TMA engine; lane 0 then issues the store.
__device__ __forceinline__ void staging_release() {
  fence_async_smem();
  __syncwarp();
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// sigma(g) = 1 / (1 + e^-g) with one ex2.approx and one rcp.approx (no IEEE division)
__device__ __forceinline__ float sigmoid_f(float g) { return rcp_approx(1.f + __expf(-g)); }
__device__ __forceinline__ float silu_f(float g) { return g * sigmoid_f(g); }

// ---------------------------------------------------------------- NEXT-1 fused dispatch
// kEpiSwiGLUDisp runs the dispatch all-to-all (F3) INSIDE the GEMM1
// launch, so GEMM1 tiles start as their rows land instead of after the whole exchange
// ("computation-communication overlap within MoE layers"):
//   * prologue (all threads of every CTA): the counts exchange and the forward-pattern tables
//     of comm.cu's dispatch (same definitions: owner segments 128-aligned in slot order, rows
//     of a slot ordered by source rank), from which the GEMM's own group tables follow;
//   * warps 2-3 of every CTA (idle in a plain GEMM) push this rank's send rows into their
//     owners' receive rows with 16-byte peer stores, 2 KB row parts claimed in chunks from a
//     global counter (so CTAs that start late -- or never, beside another kernel -- cannot
//     hold back a transfer), zero this rank's own padding rows, and count the parts done per
//     (owner, slot) segment; the warp that completes a segment releases the arrival flag
//     arrive[slot][source] = epoch in the owner's heap;
//   * the TMA producer, before the first A box of a tile, waits for the flags of exactly the
//     sources whose rows fall into its 128 rows (+ the padding flag), then orders the async
//     proxy after the acquire.
// The kernel ends the collective like comm.cu's dispatch: data flags to every peer, wait for
// every peer's, commit the epoch -- so the next collectives see the same protocol state.
// kEpiDSwiGLUComb is the backward twin (combine_bwd inside dgrad-1): no counts exchange (the
// forward's layout record), whole-row items carrying bf16(g dy) plus the dgates dot products.
struct DispTables {
  int* rows;     // [E]     rows of expert e over all sources
  int* dst;      // [E]     receive row of this rank's first row of expert e at its owner
  int* off;      // [E+1]   this rank's send layout (exclusive scan of its counts)
  int* sg_pre;   // [E+1]   row prefix over transfer segments i (seg_owner / seg_slot order)
  int* sg_src;   // [E]
  int* sg_dst;   // [E]
  int* pad_pre;  // [E_l+1] padding rows of this rank's slots, prefix
  uint64_t* epoch;   // [1]
  int* first;        // [1] this CTA won the counts ticket
};
constexpr int kDispChunk = 16;  // row parts (2 KB each) claimed per atomic
constexpr int kDispInFlight = 4; // row parts a warp loads before storing them
// Transfer order i: slot-major (el = i / EP), owners rotated inside a slot (owner rank+1
// first, self last) -- every owner's slot 0 completes first, from all sources at once, which
// is the order GEMM1 consumes its tiles in (groups ascending); the rotation keeps the sources
// of a moment on different receivers' links.
__device__ __forceinline__ int seg_owner(int i, int me, int EP) { return (me + 1 + i % EP) % EP; }
__device__ __forceinline__ int seg_slot(int i, int EP) { return i / EP; }

__device__ __forceinline__ uint64_t* arrive_flag(const KParams& p, int q, int el, int src) {
  return reinterpret_cast<uint64_t*>(peer_base(p.comm, q) + p.arrive_off) + el * (p.comm.ep + 1) + src;
}

__device__ __forceinline__ void spin_flag(const uint64_t* f, uint64_t v, int32_t* err) {
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys(f) < v) {
    if (globaltimer_ns() - t0 > 10ull * 1000 * 1000 * 1000) {
      set_device_error(err, kDevTimeout);   // a peer never arrived: sticky fault (comm.cu)
      __threadfence_system();
      __trap();
    }
    __nanosleep(64);
  }
}

// All threads of the CTA.  Fills the GEMM group tables (s_rows/s_seg/s_tile_prefix over the
// E_l local slots), s_pre[r][el] (rows of slot el from sources < r), and t.
// EXCH (dispatch): the counts exchange first; else (combine_bwd) the count matrix is the
// forward's layout record and the dropped slots' dgates are zeroed here.
template <int TILE_M, int BN, bool EXCH>
__device__ void disp_prologue(const KParams& p, const DispTables& t, int* s_rows, int* s_seg,
                              int* s_tile_prefix, int* s_pre, int* s_arrived) {
  const CommArgs& a = p.comm;
  const int E = a.E, EP = a.ep, E_l = a.E_l, me = a.rank;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    *t.epoch = *reinterpret_cast<volatile const uint64_t*>(a.epoch_ptr) + 1;
    *t.first = EXCH ? atomicAdd(p.work + 1, 1) == 0 : 0;
  }
  __syncthreads();
  const uint64_t epoch = *t.epoch;
  if (!EXCH) {
    const int64_t n = a.T * a.k;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      if (p.cb_dest_row[i] < 0) p.cb_dgates[i] = 0.f;
  }
  if (EXCH && *t.first) {   // counts exchange: this rank's row of every peer's count matrix
    for (int i = threadIdx.x; i < EP * E; i += blockDim.x) {
      const int q = i / E, e = i % E;
      reinterpret_cast<int32_t*>(peer_base(a, q) + a.countmat_off)[me * E + e] = p.disp_counts[e];
    }
    __syncthreads();   // orders the block's count stores before the lanes' releases
    if (threadIdx.x < EP)
      st_release_sys(reinterpret_cast<uint64_t*>(peer_base(a, threadIdx.x) + a.flags_off) +
                         kSlotCounts * EP + me, epoch);
  }
  if (EXCH && threadIdx.x < EP) spin_flag(a.flags + kSlotCounts * EP + threadIdx.x, epoch, a.err);
  __threadfence();
  __syncthreads();
  const int32_t* cm = EXCH ? a.countmat : p.cb_layout;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int all = 0, before = 0;
    for (int r = 0; r < EP; ++r) {
      const int c = cm[r * E + e];
      all += c;
      if (r < me) before += c;
    }
    t.rows[e] = all;
    t.dst[e] = before;
  }
  for (int el = threadIdx.x; el < E_l; el += blockDim.x) s_arrived[el] = 0;
  __syncthreads();
  for (int q = warp; q < EP; q += kThreads / 32) {   // owner q's 128-aligned slot segments
    const int32_t total = warp_scan(
        E_l,
        [&](int el) {
          const int32_t r = t.rows[a.expert_at[q * E_l + el]];
          return (r + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
        },
        [&](int el, int32_t pre) {
          if (q == me) s_seg[el] = pre;
          t.dst[a.expert_at[q * E_l + el]] += pre;
        });
    if (q == me && lane == 0) s_seg[E_l] = total;
  }
  __syncthreads();
  if (warp == 0) {          // send layout
    const int32_t total = warp_scan(
        E, [&](int e) { return cm[me * E + e]; }, [&](int e, int32_t pre) { t.off[e] = pre; });
    if (lane == 0) t.off[E] = total;
  } else if (warp == 1) {   // GEMM group tables of the local slots
    const int NT = ceil_div(p.N, BN);
    const int32_t total = warp_scan(
        E_l,
        [&](int el) {
          const int r = t.rows[a.expert_at[me * E_l + el]];
          s_rows[el] = r;
          return ceil_div(r, TILE_M) * NT;
        },
        [&](int el, int32_t pre) { s_tile_prefix[el] = pre; });
    if (lane == 0) s_tile_prefix[E_l] = total;
  } else if (warp == 2) {   // padding rows of the local slots
    const int32_t total = warp_scan(
        E_l,
        [&](int el) {
          const int r = t.rows[a.expert_at[me * E_l + el]];
          return (r + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS - r;
        },
        [&](int el, int32_t pre) { t.pad_pre[el] = pre; });
    if (lane == 0) t.pad_pre[E_l] = total;
  } else if (warp == 3) {   // receive order inside a slot: rows from sources < r
    for (int el = lane; el < E_l; el += 32) {
      const int e = a.expert_at[me * E_l + el];
      int run = 0;
      for (int r = 0; r < EP; ++r) {
        s_pre[r * E_l + el] = run;
        run += cm[r * E + e];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) {   // transfer order
    const int q = seg_owner(i, me, EP), el = seg_slot(i, EP), e = a.expert_at[q * E_l + el];
    t.sg_src[i] = t.off[e];
    t.sg_dst[i] = t.dst[e];
  }
  if (warp == 0) {
    const int32_t total = warp_scan(
        E,
        [&](int i) {
          const int e = a.expert_at[seg_owner(i, me, EP) * E_l + seg_slot(i, EP)];
          return t.off[e + 1] - t.off[e];
        },
        [&](int i, int32_t pre) { t.sg_pre[i] = pre; });
    if (lane == 0) t.sg_pre[E] = total;
  }
  if (EXCH && *t.first) {   // layout record for the later calls of this layer (as comm.cu)
    for (int i = threadIdx.x; i < EP * E; i += blockDim.x) p.disp_layout[i] = cm[i];
    for (int el = threadIdx.x; el < E_l; el += blockDim.x) p.disp_layout[EP * E + el] = s_rows[el];
    for (int el = threadIdx.x; el <= E_l; el += blockDim.x) p.disp_layout[EP * E + E_l + el] = s_seg[el];
    if (threadIdx.x == 0 && s_seg[E_l] > p.rows_cap) set_device_error(a.err, kDevOverflow);
  }
  __syncthreads();
}

// Warps 2-3: the transfer (see above), then the end of the collective.  COMB (combine_bwd):
// items are whole rows -- send-layout row r of slot (t, j) carries bf16(g[t,j] * dy[t]) and
// yields dgates[t,j] = <dy[t], ys[r]> (combine_bwd_vec, the transfer kernel's arithmetic).
constexpr int kCombChunk = 4;   // rows claimed per atomic (combine_bwd)
template <bool COMB>
__device__ void disp_copy(const KParams& p, const DispTables& t, const int* s_rows,
                          const int* s_seg) {
  const CommArgs& a = p.comm;
  const int E = a.E, EP = a.ep, E_l = a.E_l, me = a.rank;
  const int lane = threadIdx.x & 31;
  const uint64_t epoch = *t.epoch;
  const int nvec = a.d / 8;
  const int parts = COMB ? 1 : (nvec + 127) / 128;
  const int64_t row_bytes = static_cast<int64_t>(a.d) * 2;
  const int n_pad = t.pad_pre[E_l] * parts;
  const int n_items = n_pad + t.sg_pre[E] * parts;
  int32_t* segcnt = p.work + 4;
  char* xr_local = peer_base(a, me) + p.disp_dst_off;
  // segment sid (< E: transfer segment, >= E: padding of slot sid - E) gained n parts
  auto flush = [&](int sid, int n) {
    __syncwarp();   // the warp's stores are ordered before lane 0's system fence
    if (lane == 0 && n > 0) {
      __threadfence_system();
      const int target = sid < E ? (t.sg_pre[sid + 1] - t.sg_pre[sid]) * parts
                                 : (t.pad_pre[sid - E + 1] - t.pad_pre[sid - E]) * parts;
      if (atomicAdd(segcnt + sid, n) + n == target) {
        __threadfence_system();
        st_release_sys(sid < E ? arrive_flag(p, seg_owner(sid, me, EP), seg_slot(sid, EP), me)
                               : arrive_flag(p, me, sid - E, EP),
                       epoch);
      }
    }
    __syncwarp();
  };
  constexpr int kChunk = COMB ? kCombChunk : kDispChunk;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(p.work, kChunk);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n_items) break;
    const int end = min(base + kChunk, n_items);
    int cur = -1, ncur = 0;
    if constexpr (COMB) {
      for (int it = base; it < end; ++it) {
        int sid;
        if (it < n_pad) {
          const int el = upper_bound_idx(t.pad_pre, E_l + 1, it);
          const int64_t row = s_seg[el] + s_rows[el] + (it - t.pad_pre[el]);
          uint4* z = reinterpret_cast<uint4*>(xr_local + row * row_bytes);
          for (int v = lane; v < nvec; v += 32) st_v4(z + v, make_uint4(0u, 0u, 0u, 0u));
          sid = E + el;
        } else {
          const int r = it - n_pad;
          const int i = upper_bound_idx(t.sg_pre, E + 1, r);
          const int within = r - t.sg_pre[i];
          const int64_t srow = t.sg_src[i] + within;
          const int tj = p.cb_slot_of_row[srow];
          const int64_t tok = tj / a.k;
          const float g = p.cb_gates[tj];
          const uint4* pdy = reinterpret_cast<const uint4*>(p.cb_dy + tok * a.d);
          const uint4* pys = reinterpret_cast<const uint4*>(p.cb_ys + srow * a.d);
          uint4* dst = reinterpret_cast<uint4*>(peer_base(a, seg_owner(i, me, EP)) + p.disp_dst_off +
                                                static_cast<int64_t>(t.sg_dst[i] + within) * row_bytes);
          float dot = 0.f;
          for (int v0 = lane; v0 < nvec; v0 += 128) {
            uint4 av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (v0 + 32 * u < nvec) {
                av[u] = ld_nc_v4(pdy + v0 + 32 * u);
                bv[u] = ld_nc_v4(pys + v0 + 32 * u);
              }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (v0 + 32 * u >= nvec) break;
              st_v4(dst + v0 + 32 * u, combine_bwd_vec(av[u], bv[u], g, dot));
            }
          }
          dot = warp_sum(dot);
          if (lane == 0) p.cb_dgates[tj] = dot;
          sid = i;
        }
        if (sid != cur) {
          flush(cur, ncur);
          cur = sid;
          ncur = 0;
        }
        ++ncur;
      }
    } else
    for (int it = base; it < end; it += kDispInFlight) {
      // kDispInFlight row parts in flight per lane (16 B x 4 each, all loads before the stores)
      uint4 v[kDispInFlight][4];
      uint4* dst[kDispInFlight];
      int v0[kDispInFlight], sid[kDispInFlight];
#pragma unroll
      for (int h = 0; h < kDispInFlight; ++h) {
        const int item = it + h;
        dst[h] = nullptr;
        v0[h] = 0;
        sid[h] = -1;
        if (item >= end) continue;
        const uint4* src = nullptr;
        int part;
        if (item < n_pad) {
          const int r = item / parts;
          part = item - r * parts;
          const int el = upper_bound_idx(t.pad_pre, E_l + 1, r);
          const int64_t row = s_seg[el] + s_rows[el] + (r - t.pad_pre[el]);
          dst[h] = reinterpret_cast<uint4*>(xr_local + row * row_bytes);
          sid[h] = E + el;
        } else {
          const int j = item - n_pad;
          const int r = j / parts;
          part = j - r * parts;
          const int i = upper_bound_idx(t.sg_pre, E + 1, r);
          const int within = r - t.sg_pre[i];
          const int q = seg_owner(i, me, EP);
          dst[h] = reinterpret_cast<uint4*>(peer_base(a, q) + p.disp_dst_off +
                                            static_cast<int64_t>(t.sg_dst[i] + within) * row_bytes);
          src = reinterpret_cast<const uint4*>(p.disp_src + static_cast<int64_t>(t.sg_src[i] + within) * a.d);
          sid[h] = i;
        }
        v0[h] = part * 128 + lane;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int vi = v0[h] + 32 * u;
          v[h][u] = make_uint4(0u, 0u, 0u, 0u);
          if (src && vi < nvec && vi < (part + 1) * 128) v[h][u] = ld_nc_v4(src + vi);
        }
      }
#pragma unroll
      for (int h = 0; h < kDispInFlight; ++h) {
        if (!dst[h]) continue;
        const int part_end = (v0[h] - lane) + 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int vi = v0[h] + 32 * u;
          if (vi < nvec && vi < part_end) st_v4(dst[h] + vi, v[h][u]);
        }
        if (sid[h] != cur) {
          flush(cur, ncur);
          cur = sid[h];
          ncur = 0;
        }
        ++ncur;
      }
    }
    flush(cur, ncur);
  }
  // both transfer warps of this CTA are done; the last CTA ends the collective
  asm volatile("bar.sync 1, 64;" ::: "memory");
  if ((threadIdx.x >> 5) == 2) {
    int last = 0;
    if (lane == 0) {
      __threadfence_system();
      last = atomicAdd(p.work + 2, 1) == static_cast<int>(gridDim.x) - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      // every row of this rank has landed at its owner: data flag to every peer, then wait for
      // every peer's (the count-matrix reuse argument of comm.cu's publish_counts needs it)
      if (lane < EP) {
        st_release_sys(reinterpret_cast<uint64_t*>(peer_base(a, lane) + a.flags_off) + kSlotData * EP + me,
                       epoch);
        spin_flag(a.flags + kSlotData * EP + lane, epoch, a.err);
      }
      __syncwarp();
      for (int i = lane; i < 4 + E + E_l; i += 32) p.work[i] = 0;   // every CTA is past its uses
      __threadfence();
      __syncwarp();
      if (lane == 0) *reinterpret_cast<volatile uint64_t*>(a.epoch_ptr) = epoch;
    }
  }
}

// TMA producer of a fused-dispatch GEMM1: before the first A box of this CTA's 128 rows
// [lo, lo + 128) of slot el, wait for the arrival flags of the sources whose rows (and of the
// padding, which this rank zeroes) intersect them.  s_arrived caches flags already seen.
__device__ __forceinline__ void disp_wait_rows(const KParams& p, int el, int lo, int rows_el,
                                               const int* s_pre, int* s_arrived, uint64_t epoch) {
  const int EP = p.comm.ep, E_l = p.comm.E_l;
  const int alig = (rows_el + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
  const int hi = min(lo + kBM, alig);
  if (lo >= hi) return;
  uint32_t need = 0;
  for (int r = 0; r < EP; ++r) {
    const int b = s_pre[r * E_l + el];
    const int e = (r + 1 < EP) ? s_pre[(r + 1) * E_l + el] : rows_el;
    if (b < e && b < hi && e > lo) need |= 1u << r;
  }
  if (rows_el < hi && rows_el < alig) need |= 1u << EP;
  need &= ~static_cast<uint32_t>(s_arrived[el]);
  if (!need) return;
  const uint64_t* f = arrive_flag(p, p.comm.rank, el, 0);
  const uint64_t t0 = globaltimer_ns();
  while (need) {
    for (int r = 0; r <= EP; ++r)
      if (((need >> r) & 1u) && ld_acquire_sys(f + r) >= epoch) {
        need &= ~(1u << r);
        s_arrived[el] |= 1 << r;
      }
    if (need) {
      if (globaltimer_ns() - t0 > 10ull * 1000 * 1000 * 1000) {
        set_device_error(p.comm.err, kDevTimeout);
        __threadfence_system();
        __trap();
      }
      __nanosleep(32);
    }
  }
  fence_async_global();   // the TMA (async proxy) reads below come after the acquire
}

// PAIR = 2: a cluster of two CTAs on one TPC runs tcgen05.mma.cta_group::2 with M = 256;
// each CTA stages its own 128 A rows and half of the B tile, the leader (rank 0) issues the
// MMAs for both, and each CTA's TMEM holds its 128 accumulator rows.
template <int BN, bool A_MN, bool B_MN, int EPI, int PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC,
                        const __grid_constant__ CUtensorMap tmX, const KParams p) {
  // PDL: the setup below (barrier init, tensor-map prefetch, TMEM allocation) touches no
  // global memory, so it runs before griddepcontrol.wait -- overlapping the previous kernel's
  // tail; every global access (group tables, operands, outputs) comes after the wait
  pdl_trigger();
  constexpr int STG = staging_boxes<EPI>();
  using C = Cfg<BN, PAIR, STG, extra_smem<EPI>()>;
  constexpr bool DISP = (EPI == kEpiSwiGLUDisp);
  constexpr bool COMB = (EPI == kEpiDSwiGLUComb);
  constexpr bool XFER = DISP || COMB;      // a transfer fused in front of the GEMM
  constexpr bool SWIGLU = (EPI == kEpiSwiGLU || DISP);
  constexpr bool DSW = (EPI == kEpiDSwiGLU || COMB);
  constexpr bool KGROUPED = (EPI == kEpiF32Group);
  constexpr int TILE_M = kBM * PAIR;
  constexpr uint32_t IDESC = idesc_bf16(TILE_M, BN, A_MN, B_MN);
  const uint32_t rank = (PAIR == 2) ? cluster_ctarank() : 0u;
  const int tile0 = blockIdx.x / PAIR, tile_step = gridDim.x / PAIR;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStage = smem + C::RING;  // 4 x STG x 4 KB, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 4 * STG * kStageBox);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* abar = tempty + 2;   // dSwiGLU: one per epilogue warp, its G / U box loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(abar + 4);
  int* s_tile_prefix = reinterpret_cast<int*>(tmem_slot + 4);  // [kMaxGroups+1]
  int* s_seg = s_tile_prefix + kMaxGroups + 1;                   // [kMaxGroups+1]
  int* s_rows = s_seg + kMaxGroups + 1;                          // [kMaxGroups]
  int* s_pre = s_rows + kMaxGroups;                              // scatter: [EP][E_l] (<= 256)
  int* s_soff = s_pre + kMaxGroups;                              // scatter: [EP][E_l]
  // XFER: s_soff holds the arrival cache; the transfer tables follow
  DispTables dt;
  if constexpr (XFER) {
    int* q = s_soff + kMaxGroups;
    dt.epoch = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(q) + 7) & ~uintptr_t(7));
    dt.first = reinterpret_cast<int*>(dt.epoch + 1);
    dt.rows = dt.first + 1;
    dt.dst = dt.rows + kMaxGroups;
    dt.off = dt.dst + kMaxGroups;
    dt.sg_pre = dt.off + kMaxGroups + 1;
    dt.sg_src = dt.sg_pre + kMaxGroups + 1;
    dt.sg_dst = dt.sg_src + kMaxGroups;
    dt.pad_pre = dt.sg_dst + kMaxGroups;
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_groups = p.n_groups;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if (DSW) tma_prefetch_desc(&tmX);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], PAIR);     // leader: one arrival per producer of the pair
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * PAIR);  // leader: the epilogue warps of both CTAs
    }
    for (int a = 0; a < 4; ++a) mbar_init(&abar[a], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if (PAIR == 2) {
      tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, C::TMEM_COLS);
      tmem_relinquish();
    }
  }
  pdl_wait();   // the previous kernel's outputs (this launch's inputs) are complete and visible
  if constexpr (XFER) {
    disp_prologue<TILE_M, BN, DISP>(p, dt, s_rows, s_seg, s_tile_prefix, s_pre, s_soff);
  } else {
  // ---- group tables: seg_base = 128-aligned prefix of rows; tile prefix
  if (warp == 3) {
    const int NT = ceil_div(p.N, BN);
    const int MT = ceil_div(p.M, TILE_M);
    int seg_carry = 0, tile_carry = 0;
    for (int base = 0; base < n_groups; base += 32) {
      int g = base + lane;
      int rows = (g < n_groups) ? p.group_rows[g] : 0;
      int seg_sz = ((rows + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS) * MOE_ALIGN_ROWS;
      int tiles = (g < n_groups && g >= p.group_begin)
                      ? (KGROUPED ? MT * NT : ceil_div(rows, TILE_M) * NT) : 0;
      int a = seg_sz, b = tiles;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int ya = __shfl_up_sync(0xffffffffu, a, o);
        int yb = __shfl_up_sync(0xffffffffu, b, o);
        if (lane >= o) { a += ya; b += yb; }
      }
      if (g < n_groups) {
        s_rows[g] = rows;
        s_seg[g] = seg_carry + a - seg_sz;
        s_tile_prefix[g] = tile_carry + b - tiles;
      }
      seg_carry += __shfl_sync(0xffffffffu, a, 31);
      tile_carry += __shfl_sync(0xffffffffu, b, 31);
    }
    if (lane == 0) {
      s_seg[n_groups] = seg_carry;
      s_tile_prefix[n_groups] = tile_carry;
    }
  }
  if (warp == 2) {
    if (EPI == kEpiBF16 && p.scatter) {
      // reverse-pattern tables of the local experts (same definitions as comm.cu):
      //   pre[r][el]  = rows of expert (rank*E_l + el) from sources < r  (receive order)
      //   soff[r][el] = send-layout offset of that expert on source r
      const CommArgs& a = p.comm;
      const int32_t* cm = p.scatter_layout;
      for (int el = lane; el < a.E_l; el += 32) {
        const int e = a.expert_at[a.rank * a.E_l + el];  // expert in my slot el
        int run = 0;
        for (int r = 0; r < a.ep; ++r) {
          s_pre[r * a.E_l + el] = run;
          run += cm[r * a.E + e];
        }
      }
      if (lane < a.ep) {  // source `lane`'s send layout: experts in global order
        int run = 0;
        for (int e = 0; e < a.E; ++e) {
          const int slot = a.place[e];
          if (slot / a.E_l == a.rank) s_soff[lane * a.E_l + slot % a.E_l] = run;
          run += cm[lane * a.E + e];
        }
      }
    }
  }
  }  // !XFER
  tc_fence_before();
  if (PAIR == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = s_tile_prefix[n_groups];
  // Persistent schedule: cluster c takes tiles c, c + n_c, c + 2 n_c, ... of the raster
  // (decode_tile); every role walks the same sequence.  (A dynamic scheduler -- tiles from a
  // global atomic counter through a cluster queue -- was measured equal at N = 1 and 4 %
  // slower at N = 4, profiles/r02/sched/.)
  auto next_tile = [&](int w) -> int {
    const int t = tile0 + w * tile_step;
    return t < total_tiles ? t : -1;
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = 0;; ++w) {
        const int t = next_tile(w);
        if (t < 0) break;
        const Tile tl = decode_tile<KGROUPED, BN, TILE_M>(t, s_tile_prefix, s_seg, s_rows,
                                                          n_groups, p);
        if constexpr (XFER)
          disp_wait_rows(p, tl.g, tl.m * TILE_M + static_cast<int>(rank) * kBM, tl.rows_g, s_pre,
                         s_soff, *dt.epoch);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint32_t bar_addr = smem_u32(&full[stage]);
          if (PAIR == 2) {
            bar_addr = mapa_shared(bar_addr, 0);  // completion goes to the leader's barrier
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], PAIR * C::STAGE_BYTES);
            else mbar_arrive_cluster_relaxed(bar_addr);
          } else {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          }
          auto load = [&](void* dst, const CUtensorMap* tm, int c0, int c1) {
            if (PAIR == 2) tma_load_2d_pair(dst, tm, bar_addr, c0, c1);
            else tma_load_2d(dst, tm, &full[stage], c0, c1);
          };
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int m_row = tl.m * TILE_M + static_cast<int>(rank) * kBM;  // this CTA's A rows
          // ---- A
          if (A_MN) {  // K-grouped wgrad: A[m, k] stored [k rows, m cols]
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              load(a_dst + i * 8192, &tmA, m_row + i * 64, tl.seg + kb * kBK);
          } else {
            // A pair tile may reach past its group's 128-aligned segment (the tail tile of an
            // expert): this CTA's 128 rows then belong to the NEXT segment and are discarded
            // by the epilogue.  Load them out of bounds instead -- TMA zero-fills the box
            // without touching L2/HBM, and the wasted MMAs run on zero operands (less energy
            // under the power cap).
            const bool past = m_row >= ((tl.rows_g + kBM - 1) / kBM) * kBM;
            load(a_dst, &tmA, kb * kBK, past ? (1 << 30) : tl.seg + m_row);
          }
          // ---- B (a pair splits it along N: rank r holds columns [r*BN/2, (r+1)*BN/2))
          constexpr int BNC = BN / PAIR;
          if (B_MN) {
            const int krow = KGROUPED ? (tl.seg + kb * kBK)
                                      : static_cast<int>(tl.g * p.b_group_stride) + kb * kBK;
#pragma unroll
            for (int i = 0; i < BNC / 64; ++i)
              load(b_dst + i * 8192, &tmB, tl.n * BN + static_cast<int>(rank) * BNC + i * 64, krow);
          } else if (SWIGLU) {
            const int r0 = static_cast<int>(tl.g * p.b_group_stride) + tl.n * (BN / 2);
            if (PAIR == 2) {  // rank 0: W_gate rows (acc cols [0,BN/2)), rank 1: W_up rows
              load(b_dst, &tmB, kb * kBK, r0 + (rank ? static_cast<int>(p.b_split) : 0));
            } else {
              load(b_dst, &tmB, kb * kBK, r0);
              load(b_dst + (BN / 2) * 128, &tmB, kb * kBK, r0 + static_cast<int>(p.b_split));
            }
          } else {
            load(b_dst, &tmB, kb * kBK,
                 static_cast<int>(tl.g * p.b_group_stride) + tl.n * BN + static_cast<int>(rank) * BNC);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (the leader CTA of a pair) =====================
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = 0;; ++w) {
        const int t = next_tile(w);
        if (t < 0) break;
        const Tile tl = decode_tile<KGROUPED, BN, TILE_M>(t, s_tile_prefix, s_seg, s_rows,
                                                          n_groups, p);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_STRIDE;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t adesc = A_MN ? sdesc_sw128(a_base + kk * 2048, 8192, 1024)
                                        : sdesc_sw128(a_base + kk * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? sdesc_sw128(b_base + kk * 2048, 8192, 1024)
                                        : sdesc_sw128(b_base + kk * 32, 16, 1024);
            const uint32_t accum = (kb != 0 || kk != 0) ? 1u : 0u;
            if (PAIR == 2) umma_bf16_pair(d_tmem, adesc, bdesc, IDESC, accum);
            else umma_bf16(d_tmem, adesc, bdesc, IDESC, accum);
          }
          // frees the smem slot (in both CTAs of a pair) when these MMAs complete
          if (PAIR == 2) umma_commit_pair(&empty[stage], 0x3);
          else umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (tl.nkb > 0) {
          if (PAIR == 2) umma_commit_pair(&tfull[acc], 0x3);
          else umma_commit(&tfull[acc]);
        } else {
          mbar_arrive(&tfull[acc]);
          if (PAIR == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tfull[acc]), 1));
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (XFER && warp < 4) {
    // ===================== fused transfer (warps 2-3) =====================
    if constexpr (XFER) disp_copy<COMB>(p, dt, s_rows, s_seg);
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // TMEM lane quadrant ew*32 .. ew*32+31
    const uint32_t row_addr = smem_u32(sStage + ew * STG * kStageBox) + lane * 128;
    const void* box = sStage + ew * STG * kStageBox;
    int sbuf = 0;   // STG = 2: the staging box the next chunk uses
    uint32_t aph = 0;   // dSwiGLU: parity of this warp's G / U box barrier
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = 0;; ++w) {
      const int t = next_tile(w);
      if (t < 0) break;
      const Tile tl = decode_tile<KGROUPED, BN, TILE_M>(t, s_tile_prefix, s_seg, s_rows,
                                                        n_groups, p);
      const int m_box = tl.m * TILE_M + static_cast<int>(rank) * kBM + ew * 32;  // warp's 1st row
      const int mi = m_box + lane;  // row of this thread inside its group
      const bool valid = KGROUPED ? true : (mi < tl.rows_g);
      const int row0 = KGROUPED ? m_box : (tl.seg + m_box);
      // A 256-row pair tile may end past the group's 128-aligned segment: those rows belong to
      // the next group and are not written here (whole 32-row boxes, segments are 128-aligned).
      const bool box_in = KGROUPED || m_box < ((tl.rows_g + kBM - 1) / kBM) * kBM;
      const int64_t grow = static_cast<int64_t>(tl.seg) + mi;
      if (DSW && valid && grow < p.rows_cap) {
        // warm L2 with this row's saved G and U segments while the MMAs run
        const uint16_t* a = reinterpret_cast<const uint16_t*>(p.aux) + grow * p.ld_aux + tl.n * BN;
        prefetch_l2_bulk(a, BN * 2);
        prefetch_l2_bulk(a + p.f, BN * 2);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tacc =
          tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * C::ACC_STRIDE;
      if (box_in) {
      if (SWIGLU) {
        // acc cols [0, BN/2) = G, [BN/2, BN) = U for f-columns n*BN/2 ...; write G, U, H
#pragma unroll 1
        for (int c0 = 0; c0 < BN / 2; c0 += 64) {
          uint32_t ga[32], gb[32], ua[32], ub[32], w[32];
          tmem_ld32(tacc + c0, ga);
          tmem_ld32(tacc + c0 + 32, gb);
          tmem_ld32(tacc + BN / 2 + c0, ua);
          tmem_ld32(tacc + BN / 2 + c0 + 32, ub);
          tmem_ld_wait();
          if (!valid) {
#pragma unroll
            for (int q = 0; q < 32; ++q) ga[q] = gb[q] = ua[q] = ub[q] = 0u;
          }
          const int col = tl.n * (BN / 2) + c0;
#pragma unroll
          for (int part = 0; part < 3; ++part) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float x0, x1, y0, y1;
              if (part == 0) {
                x0 = __uint_as_float(ga[2 * q]); x1 = __uint_as_float(ga[2 * q + 1]);
                y0 = __uint_as_float(gb[2 * q]); y1 = __uint_as_float(gb[2 * q + 1]);
              } else if (part == 1) {
                x0 = __uint_as_float(ua[2 * q]); x1 = __uint_as_float(ua[2 * q + 1]);
                y0 = __uint_as_float(ub[2 * q]); y1 = __uint_as_float(ub[2 * q + 1]);
              } else {  // H = silu(G) * U from the fp32 accumulators
                x0 = silu_f(__uint_as_float(ga[2 * q])) * __uint_as_float(ua[2 * q]);
                x1 = silu_f(__uint_as_float(ga[2 * q + 1])) * __uint_as_float(ua[2 * q + 1]);
                y0 = silu_f(__uint_as_float(gb[2 * q])) * __uint_as_float(ub[2 * q]);
                y1 = silu_f(__uint_as_float(gb[2 * q + 1])) * __uint_as_float(ub[2 * q + 1]);
              }
              w[q] = pack_bf16(x0, x1);
              w[16 + q] = pack_bf16(y0, y1);
            }
            staging_acquire(lane);
            stage_row(row_addr, lane, w);
            staging_release();
            if (lane == 0) {
              tma_store_2d(&tmC, box, col + part * p.f, row0);
              bulk_commit();
            }
          }
        }
      } else if (EPI == kEpiBF16) {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 64) {
          uint32_t a[32], b[32], w[32];
          tmem_ld32(tacc + c0, a);
          tmem_ld32(tacc + c0 + 32, b);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            w[q] = valid ? pack_bf16(__uint_as_float(a[2 * q]), __uint_as_float(a[2 * q + 1])) : 0u;
            w[16 + q] = valid ? pack_bf16(__uint_as_float(b[2 * q]), __uint_as_float(b[2 * q + 1])) : 0u;
          }
          if (p.scatter) {
            // fused reverse all-to-all: this row's 128 bytes go straight to its source rank's
            // buffer as one asynchronous bulk copy (NVSwitch for remote ranks), so the NVLink
            // latency is absorbed by the copy engine, not by the epilogue warps
            bulk_wait_read0();                       // my previous copy has read my row
            const uint32_t lin = smem_u32(box) + lane * 128;   // linear (unswizzled) row
#pragma unroll
            for (int v = 0; v < 8; ++v)
              st_shared_v4(lin + v * 16, w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
            fence_async_smem();
            if (valid) {
              const int E_l = p.comm.E_l, g = tl.g;
              int r = 0;
              while (r + 1 < p.comm.ep && s_pre[(r + 1) * E_l + g] <= mi) ++r;
              const int64_t drow = s_soff[r * E_l + g] + (mi - s_pre[r * E_l + g]);
              bulk_copy_s2g(peer_base(p.comm, r) + p.scatter_off + (drow * p.N + tl.n * BN + c0) * 2,
                            lin, 128);
              bulk_commit();
            }
          } else {
            staging_acquire(lane);
            stage_row(row_addr, lane, w);
            staging_release();
            if (lane == 0) {
              tma_store_2d(&tmC, box, tl.n * BN + c0, row0);
              bulk_commit();
            }
          }
        }
      } else if (DSW) {
        // acc = dH for f-columns n*BN ...; dG = dH*U*silu'(G), dU = dH*silu(G) -> dgu
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 64) {
          const int col = tl.n * BN + c0;
          // the last tile of an f that is an odd multiple of 128 is half past f: those
          // accumulator columns are zero (B loaded out of bounds) and have no dG/dU columns
          if (col >= p.f) break;
          uint32_t a[32], b[32], gw[32], uw[32], w[32];
          tmem_ld32(tacc + c0, a);
          tmem_ld32(tacc + c0 + 32, b);
          if (p.aux_tma) {
            // G and U boxes [32 rows x 64 cols] through this warp's staging box by TMA (one
            // instruction each instead of 16 per-lane 16-byte loads; out-of-range rows load as
            // zeros), read back row-per-lane from the 128B-swizzled layout
            uint32_t* dst[2] = {gw, uw};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              staging_acquire(lane);   // the last TMA store from the box has read it
              if (lane == 0) {
                mbar_arrive_expect_tx(&abar[ew], kStageBox);
                tma_load_2d(const_cast<void*>(box), &tmX, &abar[ew], col + h * p.f, row0);
              }
              mbar_wait(&abar[ew], aph);
              aph ^= 1u;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                ld_shared_v4(row_addr + ((j ^ (lane & 7)) << 4), dst[h][4 * j], dst[h][4 * j + 1],
                             dst[h][4 * j + 2], dst[h][4 * j + 3]);
              __syncwarp();
            }
          } else if (valid && grow < p.rows_cap) {
            const uint16_t* src = reinterpret_cast<const uint16_t*>(p.aux) + grow * p.ld_aux + col;
            const uint4* pg = reinterpret_cast<const uint4*>(src);
            const uint4* pu = reinterpret_cast<const uint4*>(src + p.f);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const uint4 g4 = pg[v], u4 = pu[v];
              gw[4 * v] = g4.x; gw[4 * v + 1] = g4.y; gw[4 * v + 2] = g4.z; gw[4 * v + 3] = g4.w;
              uw[4 * v] = u4.x; uw[4 * v + 1] = u4.y; uw[4 * v + 2] = u4.z; uw[4 * v + 3] = u4.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) gw[q] = uw[q] = 0u;
          }
          tmem_ld_wait();
          uint32_t wu[32];  // dU words; w holds the dG words
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            // packed word q holds columns 2q, 2q+1 of the 64-column chunk
            const float dh0 = __uint_as_float(q < 16 ? a[2 * q] : b[2 * q - 32]);
            const float dh1 = __uint_as_float(q < 16 ? a[2 * q + 1] : b[2 * q - 31]);
            const float g0 = bf16_lo(gw[q]), g1 = bf16_hi(gw[q]);
            const float s0 = sigmoid_f(g0), s1 = sigmoid_f(g1);
            const float dg0 = dh0 * bf16_lo(uw[q]) * s0 * (1.f + g0 * (1.f - s0));
            const float dg1 = dh1 * bf16_hi(uw[q]) * s1 * (1.f + g1 * (1.f - s1));
            w[q] = valid ? pack_bf16(dg0, dg1) : 0u;
            wu[q] = valid ? pack_bf16(dh0 * g0 * s0, dh1 * g1 * s1) : 0u;
          }
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            staging_acquire(lane);
            if (part == 0) stage_row(row_addr, lane, w);
            else stage_row(row_addr, lane, wu);
            staging_release();
            if (lane == 0) {
              tma_store_2d(&tmC, box, col + part * p.f, row0);
              bulk_commit();
            }
          }
        }
      } else if (EPI == kEpiF32Group) {
        // wgrad: fp32 [M, N] of group g; 3-D tensor map {N, M, G} clips rows >= M per group
        if (!(tl.nkb == 0 && p.accumulate)) {
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t a[32];
            if (tl.nkb > 0) {
              tmem_ld32(tacc + c0, a);
              tmem_ld_wait();
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q) a[q] = 0u;
            }
            // the store that last used THIS box must have read it (STG = 2: that is the one
            // before the most recent; STG = 1: the most recent)
            if (lane == 0) {
              if (STG == 2) bulk_wait_read1();
              else bulk_wait_read0();
            }
            __syncwarp();
            const uint32_t off = static_cast<uint32_t>(sbuf * kStageBox);
            stage_row(row_addr + off, lane, a);
            staging_release();
            if (lane == 0) {
              const void* b = static_cast<const uint8_t*>(box) + off;
              if (p.accumulate) tma_reduce_add_3d(&tmC, b, tl.n * BN + c0, row0, tl.g);
              else tma_store_3d(&tmC, b, tl.n * BN + c0, row0, tl.g);
              bulk_commit();
            }
            sbuf ^= (STG - 1);
          }
        }
      } else {  // kEpiF32Rows: router logits / router dgrad, fp32 [rows, N] (+ bias) (+= old)
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t a[32];
          tmem_ld32(tacc + c0, a);
          tmem_ld_wait();
          const int col0 = tl.n * BN + c0;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            float v = __uint_as_float(a[q]);
            if (p.bias && col0 + q < p.N) v += p.bias[col0 + q];
            a[q] = valid ? __float_as_uint(v) : 0u;
          }
          if (p.direct_store) {
            if (valid && grow < p.rows_cap) {
              float* o = reinterpret_cast<float*>(p.out) + grow * p.ld_out;
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (col0 + q < p.N)
                  o[col0 + q] = p.accumulate ? o[col0 + q] + __uint_as_float(a[q]) : __uint_as_float(a[q]);
            }
          } else {
            staging_acquire(lane);
            stage_row(row_addr, lane, a);
            staging_release();
            if (lane == 0) {
              if (p.accumulate) tma_reduce_add_2d(&tmC, box, col0, row0);
              else tma_store_2d(&tmC, box, col0, row0);
              bulk_commit();
            }
          }
        }
      }
      }  // box_in
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR == 2 && rank != 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (EPI == kEpiBF16 && p.scatter) {
      bulk_wait0();            // every lane's row copies complete ...
      fence_async_global();    // ... and ordered before the flag release below
      __threadfence_system();
    } else if (lane == 0) {
      bulk_wait0();            // all TMA stores of this warp complete before exit
    }
  }

  tc_fence_before();
  if (PAIR == 2) cluster_sync(); else __syncthreads();
  if (EPI == kEpiBF16 && p.scatter && threadIdx.x == 0) {
    // the last CTA to finish publishes the epoch to every rank (as comm.cu's signal_done)
    const CommArgs& a = p.comm;
    if (atomicAdd(a.done, 1) == static_cast<int>(gridDim.x) - 1) {
      a.done[0] = 0;
      // device-resident epoch: advanced only by the wait_flags launch that follows
      const uint64_t epoch = *reinterpret_cast<volatile const uint64_t*>(a.epoch_ptr) + 1;
      __threadfence_system();
      for (int q = 0; q < a.ep; ++q)
        st_release_sys(reinterpret_cast<uint64_t*>(peer_base(a, q) + a.flags_off) +
                           kSlotData * a.ep + a.rank,
                       epoch);
    }
  }
  if (warp == 2) {
    tc_fence_after();
    if (PAIR == 2) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// rank-2/3 tensor map, dims innermost first, strides in bytes for dims 1..rank-1
bool make_tmap(CUtensorMap* tm, CUtensorMapDataType dt, int rank, const void* ptr,
               const int64_t* dims, const int64_t* strides, const int* box) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    if (dims[i] <= 0) return false;
    d[i] = static_cast<cuuint64_t>(dims[i]);
    b[i] = static_cast<cuuint32_t>(box[i]);
  }
  for (int i = 0; i < rank - 1; ++i) {
    if (strides[i] % 16) return false;
    s[i] = static_cast<cuuint64_t>(strides[i]);
  }
  // L2 sector promotion of TMA reads: 256 B by default; MOE_L2_PROMOTION=0/64/128 for A/B runs
  static CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  static bool promo_read = false;
  if (!promo_read) {
    const char* e = getenv("MOE_L2_PROMOTION");
    if (e && e[0] == '0') promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
    else if (e && !strcmp(e, "64")) promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    else if (e && !strcmp(e, "128")) promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    promo_read = true;
  }
  CUresult r = fn(tm, dt, rank, const_cast<void*>(ptr), d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_bf16(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                    int box_cols, int box_rows) {
  const int64_t dims[2] = {cols, rows};
  const int64_t strides[1] = {ld * 2};
  const int box[2] = {box_cols, box_rows};
  return make_tmap(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box);
}

template <int BN, bool A_MN, bool B_MN, int EPI, int PAIR>
cudaError_t launch_impl(const GemmProblem& g, cudaStream_t stream) {
  using C = Cfg<BN, PAIR, staging_boxes<EPI>(), extra_smem<EPI>()>;
  constexpr bool SWIGLU = (EPI == kEpiSwiGLU || EPI == kEpiSwiGLUDisp);
  constexpr bool DSW = (EPI == kEpiDSwiGLU || EPI == kEpiDSwiGLUComb);
  CUtensorMap ta, tb, tc;
  // A box: K-major {64 k, 128 rows}; MN-major {64 m, 64 k}
  if (!make_tmap_bf16(&ta, g.a_ptr, g.a_rows, g.a_cols, g.a_ld, 64, A_MN ? 64 : kBM))
    return cudaErrorInvalidValue;
  const int b_box_rows = B_MN ? 64 : (SWIGLU ? BN / 2 : BN / PAIR);
  if (!make_tmap_bf16(&tb, g.b_ptr, g.b_rows, g.b_cols, g.b_ld, 64, b_box_rows))
    return cudaErrorInvalidValue;
  KParams kp;
  memset(&kp, 0, sizeof(kp));
  // output: one 32-row x 128-byte box per epilogue warp
  if (EPI == kEpiF32Group) {
    const int64_t dims[3] = {g.N, g.M, g.n_groups};
    const int64_t strides[2] = {static_cast<int64_t>(g.N) * 4, static_cast<int64_t>(g.M) * g.N * 4};
    const int box[3] = {32, 32, 1};
    if (!make_tmap(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g.out, dims, strides, box))
      return cudaErrorInvalidValue;
  } else if (EPI == kEpiF32Rows) {
    const int64_t dims[2] = {g.N, g.rows_cap};
    const int64_t strides[1] = {g.ld_out * 4};
    const int box[2] = {32, 32};
    if (!make_tmap(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g.out, dims, strides, box)) {
      kp.direct_store = 1;  // e.g. E=5 logits: pitch not 16B-aligned
      tc = ta;
    }
  } else {
    const int64_t cols = SWIGLU ? 3 * static_cast<int64_t>(g.f)
                         : DSW ? 2 * static_cast<int64_t>(g.f)
                                                : g.N;
    if (!make_tmap_bf16(&tc, g.out, g.rows_cap, cols, g.ld_out, 64, 32)) return cudaErrorInvalidValue;
  }
  // dSwiGLU: the saved G | U | H rows as 32 x 64 boxes for the epilogue's TMA loads
  CUtensorMap tx = tc;
  if (DSW) {
    static int tma_aux = -1;   // MOE_DSWIGLU_TMA=0: per-lane global loads (measurements)
    if (tma_aux < 0) {
      const char* e = getenv("MOE_DSWIGLU_TMA");
      tma_aux = (e && e[0] == '0') ? 0 : 1;
    }
    if (tma_aux && make_tmap_bf16(&tx, g.aux, g.rows_cap, 3 * static_cast<int64_t>(g.f), g.ld_aux,
                                  64, 32))
      kp.aux_tma = 1;
  }
  kp.M = g.M; kp.N = g.N; kp.K = g.K;
  kp.n_groups = g.n_groups;
  kp.group_begin = g.group_begin;
  kp.group_rows = g.group_rows;
  kp.rows_cap = g.rows_cap;
  kp.b_group_stride = g.b_group_stride;
  kp.b_split = g.b_split;
  kp.n_fastest = g.n_fastest;
  kp.out = g.out; kp.ld_out = g.ld_out;
  kp.aux = g.aux; kp.ld_aux = g.ld_aux;
  kp.bias = g.bias;
  kp.f = g.f;
  kp.accumulate = g.accumulate;
  kp.scatter = g.scatter;
  if (g.scatter) {
    if (EPI != kEpiBF16 || !g.comm || !g.scatter_layout) return cudaErrorInvalidValue;
    kp.scatter_off = g.scatter_off;
    kp.scatter_layout = g.scatter_layout;
    kp.comm = *g.comm;
  }
  if (EPI == kEpiSwiGLUDisp || EPI == kEpiDSwiGLUComb) {
    const bool comb = EPI == kEpiDSwiGLUComb;
    if (!g.comm || !g.disp_work || g.n_groups != g.comm->E_l || g.comm->E > kMaxGroups ||
        (!comb && (!g.disp_counts || !g.disp_layout)) ||
        (comb && (!g.cb_layout || (g.comm->T > 0 && (!g.cb_dy || !g.cb_gates || !g.cb_ys ||
                                                     !g.cb_dgates || !g.cb_slot_of_row ||
                                                     !g.cb_dest_row)))))
      return cudaErrorInvalidValue;
    kp.cb_dy = static_cast<const uint16_t*>(g.cb_dy);
    kp.cb_gates = g.cb_gates;
    kp.cb_ys = static_cast<const uint16_t*>(g.cb_ys);
    kp.cb_dgates = g.cb_dgates;
    kp.cb_slot_of_row = g.cb_slot_of_row;
    kp.cb_dest_row = g.cb_dest_row;
    kp.cb_layout = g.cb_layout;
    kp.comm = *g.comm;
    kp.disp_src = static_cast<const uint16_t*>(g.disp_src);
    kp.disp_counts = g.disp_counts;
    kp.disp_layout = g.disp_layout;
    kp.disp_dst_off = g.disp_dst_off;
    kp.arrive_off = g.arrive_off;
    kp.work = g.disp_work;
  }
  auto kern = grouped_gemm_kernel<BN, A_MN, B_MN, EPI, PAIR>;
  // launch state is per device (a process may drive several GPUs, one ctx each)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  if (PAIR == 1) {
    const int grid = (g.max_ctas > 0 && g.max_ctas < num_sms()) ? g.max_ctas : num_sms();
    return launch_k(kern, dim3(grid), dim3(kThreads), C::SMEM, stream, ta, tb, tc, tx, kp);
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Persistent grid = the number of CTA pairs that can be co-resident (not every SM can
  // pair: a launch of more clusters would run the excess as a second, serial wave).
  static int max_clusters[kMaxDevices] = {};
  if (max_clusters[dev] == 0) {
    cfg.gridDim = dim3(num_sms() / 2 * 2);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = num_sms() / 2;
    max_clusters[dev] = n;
    if (getenv("MOE_VERBOSE"))
      fprintf(stderr, "[libmoe] gemm<BN=%d,epi=%d> pair grid: %d co-resident clusters of 2\n", BN, EPI, n);
  }
  int clusters = max_clusters[dev];
  if (g.max_ctas > 0 && g.max_ctas / 2 < clusters) clusters = g.max_ctas / 2 > 0 ? g.max_ctas / 2 : 1;
  cfg.gridDim = dim3(2 * clusters);
  cfg.numAttrs = 1 + pdl_attr(&attr[1]);
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tx, kp);
}

}  // namespace

int num_sms() {
  static int n_of[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (n_of[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n_of[dev] = n > 0 ? n : 148;
  }
  return n_of[dev];
}

#define MOE_GEMM_CASE(BN_, AMN, BMN, EPI_)                                      \
  if (g.BN == BN_ && g.a_mn == AMN && g.b_mn == BMN && g.epi == EPI_) {          \
    if (g.pair == 2 && BN_ >= 128) return launch_impl<BN_, AMN, BMN, EPI_, (BN_ >= 128 ? 2 : 1)>(g, s); \
    return launch_impl<BN_, AMN, BMN, EPI_, 1>(g, s);                            \
  }

cudaError_t launch_grouped_gemm(const GemmProblem& g, cudaStream_t s) {
  if (g.n_groups <= 0 || g.n_groups > kMaxGroups) return cudaErrorInvalidValue;
  MOE_GEMM_CASE(256, false, false, kEpiSwiGLU)
  MOE_GEMM_CASE(128, false, false, kEpiSwiGLU)
  MOE_GEMM_CASE(256, false, false, kEpiSwiGLUDisp)
  MOE_GEMM_CASE(256, false, false, kEpiBF16)
  MOE_GEMM_CASE(128, false, false, kEpiBF16)
  MOE_GEMM_CASE(64, false, false, kEpiBF16)
  MOE_GEMM_CASE(256, false, true, kEpiBF16)
  MOE_GEMM_CASE(128, false, true, kEpiBF16)
  MOE_GEMM_CASE(64, false, true, kEpiBF16)
  MOE_GEMM_CASE(256, false, true, kEpiDSwiGLU)
  MOE_GEMM_CASE(128, false, true, kEpiDSwiGLU)
  MOE_GEMM_CASE(256, false, true, kEpiDSwiGLUComb)
  MOE_GEMM_CASE(128, false, true, kEpiDSwiGLUComb)
  MOE_GEMM_CASE(256, true, true, kEpiF32Group)
  MOE_GEMM_CASE(128, true, true, kEpiF32Group)
  MOE_GEMM_CASE(64, true, true, kEpiF32Group)
  MOE_GEMM_CASE(256, false, true, kEpiF32Rows)
  MOE_GEMM_CASE(128, false, true, kEpiF32Rows)
  MOE_GEMM_CASE(64, false, true, kEpiF32Rows)
  MOE_GEMM_CASE(256, false, false, kEpiF32Rows)
  MOE_GEMM_CASE(128, false, false, kEpiF32Rows)
  MOE_GEMM_CASE(64, false, false, kEpiF32Rows)
  MOE_GEMM_CASE(16, false, false, kEpiF32Rows)
  return cudaErrorInvalidValue;
}
#undef MOE_GEMM_CASE

}  // namespace moe
