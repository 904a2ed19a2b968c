// comm.cu -- F3/F5 dispatch/combine and their backward twins over NVSwitch.
//
// The paper's all-to-alls (PAPER.md:132 four per layer; PAPER.md:351-356 volumes) are
// implemented as direct peer stores into symmetric buffers: every rank maps every
// peer's heap (cudaIpc), so a warp can write a 16-byte vector straight into a peer's
// receive row over NVLink.  PAPER.md:134 notes the flat point-to-point all-to-all is
// bandwidth-optimal on a uniform topology; one NVSwitch box is uniform, so there is
// no hierarchical phase (HALO, is multi-node prior art).
//
// Two transfer patterns serve the four all-to-alls:
//   forward  (dispatch, combine_bwd): source send-layout rows -> owner receive rows
//   reverse  (combine, dispatch_bwd): owner receive rows -> source send-layout rows
// Completion protocol per call (epoch = a per-call counter identical on all ranks):
//   all blocks store rows -> fence.sc.sys -> block counter; the last block publishes
//   flag[dst][slot][me] = epoch with st.release.sys on every rank; a 1-block wait
//   kernel spins with ld.acquire.sys until every peer's flag reaches the epoch
//   (bounded: 10 s, then MOE_ERR_TIMEOUT in the device error word).
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

// Latency tracing (build with -DMOE_TRACE only): globaltimer stamps of the phases of the
// last dispatch call, read with moe_debug_trace (not part of the C ABI).
#ifdef MOE_TRACE
__device__ unsigned long long g_trace[64][8];   // [epoch % 64][stamp]
#define MOE_TRACE_AT(i, cond)                                                        \
  do {                                                                               \
    if ((cond) && threadIdx.x == 0) g_trace[a.epoch % 64][i] = globaltimer_ns();     \
  } while (0)
#else
#define MOE_TRACE_AT(i, cond) do {} while (0)
#endif

constexpr uint64_t kTimeoutNs = 10ull * 1000 * 1000 * 1000;
constexpr int kMaxE = 256;  // validated by the C-ABI (E <= 256)
constexpr int kDyK = 8;     // combine_bwd: slots per token handled with dy read once

__device__ __forceinline__ uint64_t* peer_flag(const CommArgs& a, int q, int slot, int src) {
  return reinterpret_cast<uint64_t*>(peer_base(a, q) + a.flags_off) + slot * a.ep + src;
}

__device__ void wait_all(const CommArgs& a, int slot);

__device__ __forceinline__ uint64_t load_epoch(const CommArgs& a) {
  return *reinterpret_cast<volatile const uint64_t*>(a.epoch_ptr) + 1;
}
// The collective is complete on this rank: publish the epoch for the next call.
__device__ __forceinline__ void commit_epoch(const CommArgs& a) {
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint64_t*>(a.epoch_ptr) = a.epoch;
}

// Last block of a transfer kernel publishes the epoch to every destination rank and then
// (wait_after) waits until every peer's rows have landed here, so the whole collective is a
// single launch: the kernel completes only when this rank's receive buffer is complete.
__device__ void signal_done(const CommArgs& a, int slot, bool wait_after) {
  __shared__ int s_last;
  // bar.sync orders the block's stores before thread 0's fence.sc.sys, which is cumulative
  // over them (the grid-barrier pattern): one system fence per block, not per thread
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const int prev = atomicAdd(a.done, 1);
    s_last = (prev == static_cast<int>(gridDim.x) - 1);
    MOE_TRACE_AT(4, s_last);
    if (s_last) {
      a.done[0] = 0;
      a.done[1] = 0;  // publish_counts ticket (every block has passed it)
    }
  }
  __syncthreads();
  // the last block's lanes 0..EP-1 release the epoch to every destination rank at once
  // (one st.release per lane, issued as one warp instruction)
  if (s_last && threadIdx.x < a.ep) st_release_sys(peer_flag(a, threadIdx.x, slot, a.rank), a.epoch);
  if (wait_after && s_last) {
    wait_all(a, slot);
    MOE_TRACE_AT(5, true);
    commit_epoch(a);   // every block read the epoch before counting itself in `done`
  }
}

// Publishes this rank's E counts into row `rank` of every peer's count matrix.  ONE buffer is
// enough (the former epoch-parity double buffer never alternated): rank r writes
// its counts of dispatch i+1 into peer q's row r only after r's dispatch i completed, which
// required q's data flag of dispatch i, which q publishes only after every block of its
// dispatch i built its tables from the count matrix -- so q has finished reading row r.
// The same argument covers the dedup pair-count matrix.  Done by whichever block of the
// launch arrives first (ticket), so it
// cannot be starved by blocks that are already spinning on the counts flags.
// With ntok (the dedup dispatch) this rank's EP pair counts go into row `rank` of every
// peer's [EP x EP] pair-count matrix under the same release.
__device__ void publish_counts(const CommArgs& a, const int32_t* counts,
                               const int32_t* ntok = nullptr) {
  __shared__ int s_first;
  if (threadIdx.x == 0) s_first = (atomicAdd(a.done + 1, 1) == 0);
  __syncthreads();
  if (!s_first) return;
  const int parity = 0;   // single buffer (see above)
  const int E = a.E, EP = a.ep;
  for (int i = threadIdx.x; i < EP * E; i += blockDim.x) {
    const int q = i / E, e = i % E;
    int32_t* dst = reinterpret_cast<int32_t*>(peer_base(a, q) + a.countmat_off) +
                   (parity * EP + a.rank) * E + e;
    *dst = counts[e];
  }
  if (ntok)
    for (int i = threadIdx.x; i < EP * EP; i += blockDim.x) {
      const int q = i / EP, q2 = i % EP;
      reinterpret_cast<int32_t*>(peer_base(a, q) + a.ntokmat_off)[(parity * EP + a.rank) * EP + q2] =
          ntok[q2];
    }
  // bar.sync orders the block's count stores before the lanes' st.release.sys (cumulative)
  __syncthreads();
  if (threadIdx.x < EP) st_release_sys(peer_flag(a, threadIdx.x, kSlotCounts, a.rank), a.epoch);
  MOE_TRACE_AT(6, true);
}

__device__ void wait_all(const CommArgs& a, int slot) {
  if (threadIdx.x < a.ep) {
    const uint64_t* f = a.flags + slot * a.ep + threadIdx.x;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(f) < a.epoch) {
      if (globaltimer_ns() - t0 > kTimeoutNs) {
        // a peer never arrived: record it and fault the kernel.  The fault is sticky, so the
        // process's next synchronising call fails instead of later steps running on an
        // incomplete receive buffer (a silent timeout corrupted every later step)
        set_device_error(a.err, kDevTimeout);
        __threadfence_system();
        __trap();
      }
      __nanosleep(64);
    }
  }
  __threadfence();
  __syncthreads();
}

// Shared prologue: per-expert tables of the forward pattern for THIS source rank, from the
// [EP x E] count matrix cm.
//   off[e]  = exclusive scan of counts_all[rank][*]  (send layout)
//   dst[e]  = row of (rank, p=0) of expert e in its owner's receive buffer
//   seg[el] = this rank's receive segments (128-aligned prefix of its experts' rows)
struct FwdTables {
  int32_t off[kMaxE + 1];
  int32_t dst[kMaxE];
  int32_t seg[kMaxE + 1];
  int32_t rows[kMaxE];
};

// Needs blockDim >= 32 (EP + 1): warps 0..EP-1 scan the owners' segments, warp EP the send
// layout (every transfer kernel runs 512 threads; a 256-thread variant broke EP = 8).
__device__ void build_fwd_tables(const CommArgs& a, const int32_t* cm, FwdTables& t) {
  const int E = a.E, EP = a.ep, E_l = a.E_l;
  // per-expert rows over all sources, and rows from sources before me
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t all = 0, before = 0;
    for (int r = 0; r < EP; ++r) {
      const int32_t c = cm[r * E + e];
      all += c;
      if (r < a.rank) before += c;
    }
    t.rows[e] = all;
    t.dst[e] = before;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < EP) {  // warp q: owner q's aligned segment prefix over its slots
    const int q = warp;
    const int32_t total = warp_scan(
        E_l,
        [&](int el) {
          const int32_t r = t.rows[a.expert_at[q * E_l + el]];
          return (r + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
        },
        [&](int el, int32_t pre) {
          if (q == a.rank) t.seg[el] = pre;
          t.dst[a.expert_at[q * E_l + el]] += pre;
        });
    if (q == a.rank && lane == 0) t.seg[E_l] = total;
  } else if (warp == EP) {  // send layout: exclusive scan of my counts
    const int32_t total = warp_scan(
        E, [&](int e) { return cm[a.rank * E + e]; }, [&](int e, int32_t pre) { t.off[e] = pre; });
    if (lane == 0) t.off[E] = total;
  }
  __syncthreads();
}

// A row of nvec 16-byte vectors is copied in parts of kPartVec vectors (2 KB, 4 per lane).
constexpr int kPartVec = 128;
__device__ __forceinline__ int row_parts(int nvec) { return (nvec + kPartVec - 1) / kPartVec; }
// One warp's share of a 2 KB row part: up to 4 x 16 B per lane.
struct PartBuf {
  uint4 v[kPartVec / 32];
};
__device__ __forceinline__ void load_part(PartBuf& b, const uint4* __restrict__ src, int nvec,
                                          int part, int lane) {
  const int v0 = part * kPartVec + lane;
#pragma unroll
  for (int i = 0; i < kPartVec / 32; ++i)
    if (v0 + 32 * i < nvec && v0 + 32 * i < (part + 1) * kPartVec) b.v[i] = ld_nc_v4(src + v0 + 32 * i);
}
__device__ __forceinline__ void store_part(uint4* dst, const PartBuf& b, int nvec, int part,
                                           int lane) {
  const int v0 = part * kPartVec + lane;
#pragma unroll
  for (int i = 0; i < kPartVec / 32; ++i)
    if (v0 + 32 * i < nvec && v0 + 32 * i < (part + 1) * kPartVec) st_v4(dst + v0 + 32 * i, b.v[i]);
}

// all four loads of a lane are issued before its stores
__device__ __forceinline__ void copy_part(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                          int nvec, int part, int lane) {
  PartBuf b;
  load_part(b, src, nvec, part, lane);
  store_part(dst, b, nvec, part, lane);
}

// Copy segments in transfer order.  Segment i moves `count` consecutive rows from
// src_base.. (local) to dst_base.. on rank dst_rank.  The order is rotated by rank
// (destination rank+1 first, self last), so at any moment the sources of an all-to-all
// write to different destinations instead of all hitting the same receiver's links.
struct SegTable {
  int32_t prefix[kMaxE + 1];
  int32_t src_base[kMaxE];
  int32_t dst_base[kMaxE];
  int32_t dst_rank[kMaxE];
  int32_t count[kMaxE];
};

// Exclusive scan of t.count[0..n) into t.prefix[0..n] (warp 0; n <= kMaxE).
__device__ void scan_segments(SegTable& t, int n) {
  if (threadIdx.x < 32) {
    const int32_t total = warp_scan(
        n, [&](int i) { return t.count[i]; }, [&](int i, int32_t pre) { t.prefix[i] = pre; });
    if (threadIdx.x == 0) t.prefix[n] = total;
  }
  __syncthreads();
}

// Row pass of combine_bwd for one slot: dot = <a, b> over the row (fp32, each lane adding its
// vectors v = lane, lane+32, ... in increasing v: the accumulation order is fixed) and, with
// dst, dst = bf16(g * a).  Four vectors of each row per lane are loaded before any is used,
// so a warp keeps 8 x 512 B in flight instead of waiting on one load pair per iteration.
__device__ __forceinline__ float dot_scale_row(const uint4* __restrict__ a,
                                               const uint4* __restrict__ b, uint4* dst, float g,
                                               int nvec, int lane) {
  float dot = 0.f;
  for (int v0 = lane; v0 < nvec; v0 += 128) {
    uint4 av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + 32 * u < nvec) {
        av[u] = ld_nc_v4(a + v0 + 32 * u);
        if (b) bv[u] = ld_nc_v4(b + v0 + 32 * u);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (v0 + 32 * u >= nvec) break;
      const uint4 o = combine_bwd_vec(av[u], b ? bv[u] : make_uint4(0u, 0u, 0u, 0u), g, dot);
      if (dst) st_v4(dst + v0 + 32 * u, o);
    }
  }
  return warp_sum(dot);
}

// Forward pattern.  mode 0: payload = src send row.  mode 1 (combine_bwd): payload of
// slot (t,j) = gates[t,j] * dy[t] (bf16), and dgates[t,j] = <dy[t], ys[dest_row[t,j]]>.
// mode 0 is the whole dispatch in one launch: counts exchange (first block), every block
// waits for all peers' counts, the first block writes the layout record, rows are stored,
// and the last block waits for every peer's rows.
template <int MODE>
__global__ void __launch_bounds__(512) forward_transfer_kernel(CommArgs a, int32_t* __restrict__ layout,
                                        const int32_t* __restrict__ counts, int64_t recv_rows_cap,
                                        const uint16_t* __restrict__ src, int64_t dst_off,
                                        uint16_t* __restrict__ local_dst,
                                        const int32_t* __restrict__ dest_row,
                                        const float* __restrict__ gates,
                                        const uint16_t* __restrict__ dy,
                                        const uint16_t* __restrict__ ys,
                                        float* __restrict__ dgates, int s0, int s1) {
  pdl_wait();
  pdl_trigger();
  __shared__ FwdTables tb;
  __shared__ SegTable sg;
  a.epoch = load_epoch(a);
  const int32_t* cm = layout;
  // the first range (s0 == 0) of a dispatch exchanges the counts and writes the layout
  // record; later ranges of the same step read the counts back from that record
  const bool exchange = (MODE == 0 && s0 == 0);
  MOE_TRACE_AT(0, MODE == 0 && blockIdx.x == 0);
  if (exchange) {
    publish_counts(a, counts);
    wait_all(a, kSlotCounts);
    MOE_TRACE_AT(1, blockIdx.x == 0);
    cm = a.countmat;
  }
  build_fwd_tables(a, cm, tb);
  if (exchange && blockIdx.x == 0) {  // layout record for the later calls of this layer
    const int EP = a.ep, E = a.E, E_l = a.E_l;
    for (int i = threadIdx.x; i < EP * E; i += blockDim.x) layout[i] = cm[i];
    for (int el = threadIdx.x; el < E_l; el += blockDim.x)
      layout[EP * E + el] = tb.rows[a.expert_at[a.rank * E_l + el]];
    for (int el = threadIdx.x; el <= E_l; el += blockDim.x) layout[EP * E + E_l + el] = tb.seg[el];
    if (threadIdx.x == 0 && tb.seg[E_l] > recv_rows_cap) set_device_error(a.err, kDevOverflow);
  }
  if (MODE == 0) {
    for (int i = threadIdx.x; i < a.E; i += blockDim.x) {
      const int q = (a.rank + 1 + i / a.E_l) % a.ep;   // rotated owner order
      const int el = i % a.E_l;
      const int e = a.expert_at[q * a.E_l + el];
      sg.count[i] = (el >= s0 && el < s1) ? tb.off[e + 1] - tb.off[e] : 0;
      sg.src_base[i] = tb.off[e];
      sg.dst_base[i] = tb.dst[e];
      sg.dst_rank[i] = q;
    }
    __syncthreads();
    scan_segments(sg, a.E);
    MOE_TRACE_AT(2, blockIdx.x == 0);
  }
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d;
  const int nvec = d / 8;
  const int64_t row_bytes = static_cast<int64_t>(d) * 2;
  const int E = a.E, E_l = a.E_l;
  // padding rows of the local receive buffer in slots [s0, s1) (zeroed every call)
  const int64_t pad_base = tb.seg[s0];
  const int64_t n_pad_rows = tb.seg[s1] - pad_base;
  // mode 0 work item = one 2 KB part of a row (a few rows still spread over many warps);
  // mode 1 = one token (its k rows and their dot products)
  const int parts = (MODE == 0) ? row_parts(nvec) : 1;
  const int64_t n_items = (MODE == 0) ? static_cast<int64_t>(sg.prefix[E]) * parts : a.T;

  for (int64_t w = gwarp; w < n_items + n_pad_rows; w += nwarps) {
    if (w >= n_items) {
      const int64_t row = pad_base + (w - n_items);
      const int el = upper_bound_idx(tb.seg, E_l + 1, row);
      const int64_t within = row - tb.seg[el];
      if (within < tb.rows[a.expert_at[a.rank * E_l + el]]) continue;  // data row, not padding
      uint4* dst = reinterpret_cast<uint4*>(local_dst + row * d);
      for (int v = lane; v < nvec; v += 32) dst[v] = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    if (MODE == 0) {
      const int64_t r = w / parts;
      const int part = static_cast<int>(w - r * parts);
      const int i = upper_bound_idx(sg.prefix, E + 1, r);
      const int64_t within = r - sg.prefix[i];
      const int64_t row = sg.src_base[i] + within;
      const int64_t drow = sg.dst_base[i] + within;
      uint4* dst = reinterpret_cast<uint4*>(peer_base(a, sg.dst_rank[i]) + dst_off + drow * row_bytes);
      copy_part(dst, reinterpret_cast<const uint4*>(src + row * d), nvec, part, lane);
    } else if (a.k <= kDyK) {
      // one token: dy is read ONCE per 2 KB part for all its slots (the slot loop runs inside
      // the part loop), each slot's ys part once; lane vectors are visited in increasing v
      // as in dot_scale_row, so dgates are identical to the per-slot path
      const int64_t t = w;
      const int k = static_cast<int>(a.k);
      uint4* dstp[kDyK];
      const uint4* ysp[kDyK];
      float gj[kDyK], dot[kDyK];
#pragma unroll
      for (int j = 0; j < kDyK; ++j) {
        dstp[j] = nullptr;
        ysp[j] = nullptr;
        gj[j] = 0.f;
        dot[j] = 0.f;
        if (j >= k) continue;
        const int32_t row = dest_row[t * k + j];
        if (row < 0) {
          if (lane == 0 && s0 == 0) dgates[t * k + j] = 0.f;
          continue;
        }
        const int e = upper_bound_idx(tb.off, E + 1, row);
        const int slot = a.place[e] % E_l;
        if (slot < s0 || slot >= s1) continue;   // another range's row
        const int q = a.place[e] / E_l;
        const int64_t drow = tb.dst[e] + (row - tb.off[e]);
        dstp[j] = reinterpret_cast<uint4*>(peer_base(a, q) + dst_off + drow * row_bytes);
        ysp[j] = reinterpret_cast<const uint4*>(ys + static_cast<int64_t>(row) * d);
        gj[j] = gates[t * k + j];
      }
      const uint4* pdy = reinterpret_cast<const uint4*>(dy + t * d);
      for (int v0 = lane; v0 < nvec; v0 += 128) {
        uint4 av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + 32 * u < nvec) av[u] = ld_nc_v4(pdy + v0 + 32 * u);
#pragma unroll
        for (int j = 0; j < kDyK; ++j) {
          if (ysp[j] == nullptr) continue;
          uint4 bv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (v0 + 32 * u < nvec) bv[u] = ld_nc_v4(ysp[j] + v0 + 32 * u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (v0 + 32 * u >= nvec) break;
            st_v4(dstp[j] + v0 + 32 * u, combine_bwd_vec(av[u], bv[u], gj[j], dot[j]));
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kDyK; ++j) {
        if (ysp[j] == nullptr) continue;
        const float v = warp_sum(dot[j]);
        if (lane == 0) dgates[t * k + j] = v;
      }
    } else {
      const int64_t t = w;
      for (int j = 0; j < a.k; ++j) {
        const int32_t row = dest_row[t * a.k + j];
        if (row < 0) {
          if (lane == 0 && s0 == 0) dgates[t * a.k + j] = 0.f;
          continue;
        }
        const int e = upper_bound_idx(tb.off, E + 1, row);
        const int slot = a.place[e] % E_l;
        if (slot < s0 || slot >= s1) continue;   // another range's row
        const float g = gates[t * a.k + j];
        const int q = a.place[e] / E_l;
        const int64_t drow = tb.dst[e] + (row - tb.off[e]);
        uint4* dst = reinterpret_cast<uint4*>(peer_base(a, q) + dst_off + drow * row_bytes);
        const float dot = dot_scale_row(reinterpret_cast<const uint4*>(dy + t * d),
                                        reinterpret_cast<const uint4*>(ys + static_cast<int64_t>(row) * d),
                                        dst, g, nvec, lane);
        if (lane == 0) dgates[t * a.k + j] = dot;
      }
    }
  }
  MOE_TRACE_AT(3, MODE == 0 && blockIdx.x == 0);
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// Reverse pattern: owner receive rows -> the same send-layout row on the source.
__global__ void __launch_bounds__(512) reverse_transfer_kernel(CommArgs a, const int32_t* __restrict__ layout,
                                        const uint16_t* __restrict__ src, int64_t dst_off) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_seg[kMaxE + 1];
  __shared__ int32_t s_pre[MOE_MAX_EP][kMaxE];   // rows of my slot el's expert from sources < r
  __shared__ int32_t s_soff[MOE_MAX_EP][kMaxE];  // send-layout offset of that expert on source r
  a.epoch = load_epoch(a);
  const int E = a.E, EP = a.ep, E_l = a.E_l;
  const int32_t* cm = layout;
  for (int i = threadIdx.x; i <= E_l; i += blockDim.x) s_seg[i] = layout[EP * E + E_l + i];
  for (int el = threadIdx.x; el < E_l; el += blockDim.x) {
    const int e = a.expert_at[a.rank * E_l + el];
    int32_t run = 0;
    for (int r = 0; r < EP; ++r) {
      s_pre[r][el] = run;
      run += cm[r * E + e];
    }
  }
  if ((threadIdx.x >> 5) < EP) {  // warp r: source r's send layout, experts in global order
    const int r = threadIdx.x >> 5;
    warp_scan(
        E, [&](int e) { return cm[r * E + e]; },
        [&](int e, int32_t pre) {
          const int slot = a.place[e];
          if (slot / E_l == a.rank) s_soff[r][slot % E_l] = pre;
        });
  }
  __syncthreads();
  __shared__ SegTable sg;
  const int nseg = EP * E_l;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    const int r = (a.rank + 1 + i / E_l) % EP;   // rotated source order
    const int el = i % E_l;
    sg.count[i] = cm[r * E + a.expert_at[a.rank * E_l + el]];
    sg.src_base[i] = s_seg[el] + s_pre[r][el];
    sg.dst_base[i] = s_soff[r][el];
    sg.dst_rank[i] = r;
  }
  __syncthreads();
  scan_segments(sg, nseg);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d, nvec = d / 8;
  const int64_t row_bytes = static_cast<int64_t>(d) * 2;
  const int parts = row_parts(nvec);
  const int64_t n_items = static_cast<int64_t>(sg.prefix[nseg]) * parts;
  for (int64_t w = gwarp; w < n_items; w += nwarps) {
    const int64_t v = w / parts;
    const int part = static_cast<int>(w - v * parts);
    const int i = upper_bound_idx(sg.prefix, nseg + 1, v);
    const int64_t within = v - sg.prefix[i];
    const int64_t row = sg.src_base[i] + within;
    const int64_t srow = sg.dst_base[i] + within;
    uint4* dst = reinterpret_cast<uint4*>(peer_base(a, sg.dst_rank[i]) + dst_off + srow * row_bytes);
    copy_part(dst, reinterpret_cast<const uint4*>(src + row * d), nvec, part, lane);
  }
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// ---------------------------------------------------------------- NEXT-4 dedup all-to-all
// Reading R18 (oracle/dedup.py): a token whose kept slots share an owner crosses
// NVLink once per (token, owner) PAIR instead of once per slot (X-MoE's
// "redundancy-based communication bypassing").  Owner q's token
// buffer holds its pairs ordered (source r, tslot): row tok_base[q][r] + tslot with
// tok_base[q][r] = sum_{r'<r} ntok[r'][q]; source r's pair buffers hold them ordered
// (owner q, tslot): row pair_base[r][q] + tslot = pdest[t, q].

// The pair bases of this rank from the pair-count matrix nm [EP x EP]:
//   tok_base[q]  = first row of my pairs in owner q's token buffer
//   pair_base[q] = first row of owner q's pairs in my pair buffers (pdest - pair_base = tslot)
__device__ __forceinline__ void pair_bases(const CommArgs& a, const int32_t* nm, int32_t* tok_base,
                                           int32_t* pair_base) {
  const int EP = a.ep;
  if (threadIdx.x < EP) {
    const int q = threadIdx.x;
    int32_t tb = 0, pb = 0;
    for (int r = 0; r < a.rank; ++r) tb += nm[r * EP + q];
    for (int q2 = 0; q2 < q; ++q2) pb += nm[a.rank * EP + q2];
    tok_base[q] = tb;
    pair_base[q] = pb;
  }
  __syncthreads();
}

// Forward pattern, deduplicated.  Work item = (token t, 2 KB part): the part is read ONCE and
// stored to every owner t has a pair with, in rotated owner order.  MODE 0 (dispatch) also
// exchanges counts and pair counts, writes the layout and pair records, and stores each
// pair's slot lists (lane j: receive row of slot j if owned by q and kept, else -1; gate).
template <int MODE>
__global__ void __launch_bounds__(512) dedup_forward_kernel(CommArgs a, int32_t* __restrict__ layout,
                                     int32_t* __restrict__ dlayout,
                                     const int32_t* __restrict__ counts,
                                     const int32_t* __restrict__ ntok, int64_t recv_rows_cap,
                                     const uint16_t* __restrict__ src,
                                     const int32_t* __restrict__ pdest,
                                     const int32_t* __restrict__ dest_row,
                                     const int32_t* __restrict__ topk_idx,
                                     const float* __restrict__ gates, int64_t tok_off,
                                     int64_t rlist_off, int64_t glist_off,
                                     const uint16_t* __restrict__ ys, float* __restrict__ dgates) {
  pdl_wait();
  pdl_trigger();
  __shared__ FwdTables tb;
  __shared__ int32_t s_tok_base[MOE_MAX_EP], s_pair_base[MOE_MAX_EP];
  a.epoch = load_epoch(a);
  const int EP = a.ep, E = a.E, E_l = a.E_l;
  const int32_t* nm = dlayout;
  if (MODE == 0) {
    publish_counts(a, counts, ntok);
    wait_all(a, kSlotCounts);
    const int32_t* cm = a.countmat;
    nm = a.ntokmat;
    build_fwd_tables(a, cm, tb);
    if (blockIdx.x == 0) {  // layout record (as moe_dispatch) + pair record
      for (int i = threadIdx.x; i < EP * E; i += blockDim.x) layout[i] = cm[i];
      for (int el = threadIdx.x; el < E_l; el += blockDim.x)
        layout[EP * E + el] = tb.rows[a.expert_at[a.rank * E_l + el]];
      for (int el = threadIdx.x; el <= E_l; el += blockDim.x) layout[EP * E + E_l + el] = tb.seg[el];
      for (int i = threadIdx.x; i < EP * EP; i += blockDim.x) dlayout[i] = nm[i];
      if (threadIdx.x == 0 && tb.seg[E_l] > recv_rows_cap) set_device_error(a.err, kDevOverflow);
    }
  }
  pair_bases(a, nm, s_tok_base, s_pair_base);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d, nvec = d / 8, k = static_cast<int>(a.k);
  const int64_t row_bytes = static_cast<int64_t>(d) * 2;
  const int parts = row_parts(nvec);
  const int64_t n_items = a.T * parts;
  // MODE 1 with ys: T more items, dgates[t,j] = <dy[t], ys[dest_row[t,j]]> at the source
  // (the fused forward leaves no O on the owner: its GEMM2 stored the rows into ys)
  const int64_t n_dot = (MODE == 1 && ys) ? a.T : 0;
  for (int64_t w = gwarp; w < n_items + n_dot; w += nwarps) {
    if (w >= n_items) {
      const int64_t t = w - n_items;
      const uint4* pdy = reinterpret_cast<const uint4*>(src + t * d);
      for (int j = 0; j < k; ++j) {
        const int32_t row = dest_row[t * k + j];
        const float dot = row < 0 ? 0.f
            : dot_scale_row(pdy, reinterpret_cast<const uint4*>(ys + static_cast<int64_t>(row) * d),
                            nullptr, 0.f, nvec, lane);
        if (lane == 0) dgates[t * k + j] = dot;
      }
      continue;
    }
    const int64_t t = w / parts;
    const int part = static_cast<int>(w - t * parts);
    const int32_t pd = lane < EP ? pdest[t * EP + lane] : -1;   // lane q: pair row for owner q
    const uint32_t mask = __ballot_sync(0xffffffffu, pd >= 0);
    if (!mask) continue;
    PartBuf b;
    load_part(b, reinterpret_cast<const uint4*>(src + t * d), nvec, part, lane);
    int32_t rr = -1, qj = -1;
    float g = 0.f;
    if (MODE == 0 && part == 0 && lane < k) {
      const int32_t dr = dest_row[t * k + lane];
      if (dr >= 0) {
        const int e = topk_idx[t * k + lane];
        qj = a.place[e] / E_l;
        rr = tb.dst[e] + (dr - tb.off[e]);
        g = gates[t * k + lane];
      }
    }
    for (int i = 0; i < EP; ++i) {
      const int q = (a.rank + 1 + i) % EP;   // rotated owner order, self last
      const int32_t pq = __shfl_sync(0xffffffffu, pd, q);
      if (!((mask >> q) & 1u)) continue;
      const int64_t u = s_tok_base[q] + (pq - s_pair_base[q]);
      char* base = peer_base(a, q);
      store_part(reinterpret_cast<uint4*>(base + tok_off + u * row_bytes), b, nvec, part, lane);
      if (MODE == 0 && part == 0 && lane < k) {
        const int32_t rl = (qj == q) ? rr : -1;
        reinterpret_cast<int32_t*>(base + rlist_off)[u * k + lane] = rl;
        reinterpret_cast<float*>(base + glist_off)[u * k + lane] = rl >= 0 ? g : 0.f;
      }
    }
  }
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// Owner, local.  MODE 0: xr[rlist[u][j]] = tok[u] (work item = (pair, 2 KB part)).
// MODE 1: dst[rl] = bf16(g * tok[u]) and dg_own[u][j] = <tok[u], O[rl]> (work item = pair).
// Both zero the padding rows of dst's receive segments.
template <int MODE>
__global__ void __launch_bounds__(512) dedup_expand_kernel(CommArgs a, const int32_t* __restrict__ layout,
                                    const int32_t* __restrict__ dlayout,
                                    const uint16_t* __restrict__ tok,
                                    const int32_t* __restrict__ rlist,
                                    const float* __restrict__ glist,
                                    const uint16_t* __restrict__ O, uint16_t* __restrict__ dst,
                                    float* __restrict__ dg_own) {
  pdl_wait();
  pdl_trigger();
  const int EP = a.ep, E = a.E, E_l = a.E_l, k = static_cast<int>(a.k);
  __shared__ int32_t s_seg[kMaxE + 1];
  __shared__ int32_t s_rows[kMaxE];
  for (int i = threadIdx.x; i <= E_l; i += blockDim.x) s_seg[i] = layout[EP * E + E_l + i];
  for (int i = threadIdx.x; i < E_l; i += blockDim.x) s_rows[i] = layout[EP * E + i];
  __syncthreads();
  int64_t n_pairs = 0;
  for (int r = 0; r < EP; ++r) n_pairs += dlayout[r * EP + a.rank];
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d, nvec = d / 8;
  const int parts = (MODE == 0) ? row_parts(nvec) : 1;
  const int64_t n_items = n_pairs * parts;
  const int64_t n_rows = s_seg[E_l];
  for (int64_t w = gwarp; w < n_items + n_rows; w += nwarps) {
    if (w >= n_items) {  // padding rows of the receive segments
      const int64_t row = w - n_items;
      const int el = upper_bound_idx(s_seg, E_l + 1, row);
      if (row - s_seg[el] < s_rows[el]) continue;
      uint4* z = reinterpret_cast<uint4*>(dst + row * d);
      for (int v = lane; v < nvec; v += 32) z[v] = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    const int64_t u = w / parts;
    const int part = static_cast<int>(w - u * parts);
    const int32_t rl_l = lane < k ? rlist[u * k + lane] : -1;
    const uint4* ptok = reinterpret_cast<const uint4*>(tok + u * d);
    if (MODE == 0) {
      PartBuf b;
      load_part(b, ptok, nvec, part, lane);
      for (int j = 0; j < k; ++j) {
        const int32_t rl = __shfl_sync(0xffffffffu, rl_l, j);
        if (rl >= 0) store_part(reinterpret_cast<uint4*>(dst + static_cast<int64_t>(rl) * d), b, nvec, part, lane);
      }
    } else {
      const float g_l = lane < k ? glist[u * k + lane] : 0.f;
      for (int j = 0; j < k; ++j) {
        const int32_t rl = __shfl_sync(0xffffffffu, rl_l, j);
        const float g = __shfl_sync(0xffffffffu, g_l, j);
        if (rl < 0) {
          if (lane == 0 && dg_own) dg_own[u * k + j] = 0.f;
          continue;
        }
        uint4* pdst = reinterpret_cast<uint4*>(dst + static_cast<int64_t>(rl) * d);
        // dO rows (and, with O, dg = <dy, O>; without O dgates were formed at the source)
        const float dot = dot_scale_row(
            ptok, O ? reinterpret_cast<const uint4*>(O + static_cast<int64_t>(rl) * d) : nullptr,
            pdst, g, nvec, lane);
        if (lane == 0 && O) dg_own[u * k + j] = dot;
      }
    }
  }
}

// Reverse pattern, deduplicated (owner -> sources).  Work item = (pair u, 2 KB part):
// part[u] = bf16( sum_j w_j rows[rlist[u][j]] ) in fp32, j ascending (MODE 0: w = glist,
// MODE 1: w = 1), stored at the source's pair row; MODE 1 also sends dg_own[u][*].  Pairs
// are visited in rotated source order.
template <int MODE>
__global__ void __launch_bounds__(512) dedup_reduce_kernel(CommArgs a, const int32_t* __restrict__ dlayout,
                                    const int32_t* __restrict__ rlist,
                                    const float* __restrict__ glist,
                                    const uint16_t* __restrict__ rows,
                                    const float* __restrict__ dg_own, int64_t part_off,
                                    int64_t dgpart_off) {
  pdl_wait();
  pdl_trigger();
  a.epoch = load_epoch(a);
  const int EP = a.ep, k = static_cast<int>(a.k);
  __shared__ int32_t s_tok_base[MOE_MAX_EP + 1];   // my token-buffer rows of source r
  __shared__ int32_t s_pb[MOE_MAX_EP];             // my pairs' first row at source r
  __shared__ int32_t s_prefix[MOE_MAX_EP + 1];     // rotated source order
  __shared__ int32_t s_src[MOE_MAX_EP];
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int r = 0; r < EP; ++r) {
      s_tok_base[r] = run;
      run += dlayout[r * EP + a.rank];
      int32_t pb = 0;
      for (int q = 0; q < a.rank; ++q) pb += dlayout[r * EP + q];
      s_pb[r] = pb;
    }
    s_tok_base[EP] = run;
    int32_t pre = 0;
    for (int i = 0; i < EP; ++i) {
      const int r = (a.rank + 1 + i) % EP;
      s_src[i] = r;
      s_prefix[i] = pre;
      pre += dlayout[r * EP + a.rank];
    }
    s_prefix[EP] = pre;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int d = a.d, nvec = d / 8;
  const int64_t row_bytes = static_cast<int64_t>(d) * 2;
  const int parts = row_parts(nvec);
  const int64_t n_items = static_cast<int64_t>(s_prefix[EP]) * parts;
  for (int64_t w = gwarp; w < n_items; w += nwarps) {
    const int64_t v = w / parts;
    const int part = static_cast<int>(w - v * parts);
    const int i = upper_bound_idx(s_prefix, EP + 1, v);
    const int r = s_src[i];
    const int64_t u = s_tok_base[r] + (v - s_prefix[i]);
    const int64_t prow = s_pb[r] + (v - s_prefix[i]);
    const int32_t rl_l = lane < k ? rlist[u * k + lane] : -1;
    const float w_l = (MODE == 0) ? (lane < k ? glist[u * k + lane] : 0.f) : 1.f;
    float acc[kPartVec / 32][8];
#pragma unroll
    for (int c = 0; c < kPartVec / 32; ++c)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[c][q] = 0.f;
    const int v0 = part * kPartVec + lane;
    const int v1 = min(nvec, (part + 1) * kPartVec);
    for (int j = 0; j < k; ++j) {
      const int32_t rl = __shfl_sync(0xffffffffu, rl_l, j);
      const float wj = __shfl_sync(0xffffffffu, w_l, j);
      if (rl < 0) continue;
      const uint4* pr = reinterpret_cast<const uint4*>(rows + static_cast<int64_t>(rl) * d);
#pragma unroll
      for (int c = 0; c < kPartVec / 32; ++c)
        if (v0 + 32 * c < v1) acc_bf16x8(acc[c], ld_nc_v4(pr + v0 + 32 * c), wj);
    }
    uint4* pdst = reinterpret_cast<uint4*>(peer_base(a, r) + part_off + prow * row_bytes);
#pragma unroll
    for (int c = 0; c < kPartVec / 32; ++c)
      if (v0 + 32 * c < v1)
        st_v4(pdst + v0 + 32 * c,
              make_uint4(pack_bf16(acc[c][0], acc[c][1]), pack_bf16(acc[c][2], acc[c][3]),
                         pack_bf16(acc[c][4], acc[c][5]), pack_bf16(acc[c][6], acc[c][7])));
    if (MODE == 1 && part == 0 && lane < k)
      reinterpret_cast<float*>(peer_base(a, r) + dgpart_off)[prow * k + lane] = dg_own[u * k + lane];
  }
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// Waits for every rank's data flag of this epoch (the GEMM-fused reverse all-to-alls).
// The GEMM that preceded it published load_epoch(a) (the counter is not advanced until here).
__global__ void wait_flags_kernel(CommArgs a, int slot) {
  pdl_wait();
  pdl_trigger();
  a.epoch = load_epoch(a);
  wait_all(a, slot);
  commit_epoch(a);
}

// NEXT-2 expert migration (reading R17): every expert whose slot changes is
// pushed by its OLD owner from its local src slot into the NEW owner's dst slot (symmetric
// buffers at the same heap offset on every rank; local slot moves are local stores).
// Protocol: the first block (ticket) announces this rank on the counts slot and every block
// waits until every peer has announced, so no peer can still be reading its dst from earlier
// stream work; then the copies; then the usual data-slot completion (the last block waits for
// every peer's stores to have landed here).  Work item = one 2 KB part of one 16-byte-vector
// "row" of kMigRowVec vectors of an expert.
constexpr int kMigRowVec = 128;
__global__ void __launch_bounds__(512) migrate_kernel(CommArgs a, MigrateList ml, const uint16_t* __restrict__ src,
                               int64_t dst_off, int64_t bytes_per_expert) {
  pdl_wait();
  pdl_trigger();
  a.epoch = load_epoch(a);
  {
    __shared__ int s_first;
    if (threadIdx.x == 0) s_first = (atomicAdd(a.done + 1, 1) == 0);
    __syncthreads();
    if (s_first && threadIdx.x < a.ep)
      st_release_sys(peer_flag(a, threadIdx.x, kSlotCounts, a.rank), a.epoch);
    wait_all(a, kSlotCounts);
  }
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nvec_e = bytes_per_expert / 16;
  const int64_t rows_e = (nvec_e + kMigRowVec - 1) / kMigRowVec;
  const int64_t n_items = static_cast<int64_t>(ml.n) * rows_e;
  for (int64_t w = gwarp; w < n_items; w += nwarps) {
    const int m = static_cast<int>(w / rows_e);
    const int64_t row = w - static_cast<int64_t>(m) * rows_e;
    const int64_t v0 = row * kMigRowVec;
    const int64_t nv = (nvec_e - v0) < kMigRowVec ? (nvec_e - v0) : kMigRowVec;
    const uint4* ps = reinterpret_cast<const uint4*>(
        reinterpret_cast<const char*>(src) + ml.src_slot[m] * bytes_per_expert) + v0;
    uint4* pd = reinterpret_cast<uint4*>(peer_base(a, ml.dst_rank[m]) + dst_off +
                                         ml.dst_slot[m] * bytes_per_expert) + v0;
    copy_part(pd, ps, static_cast<int>(nv), 0, lane);
  }
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// Equal-split all-to-all (config 5 of BASELINE.json; SPEC.md:476 transpose law): chunk q of
// this rank's send buffer -> chunk `rank` of rank q's symmetric receive buffer.  The layout is
// static, so there is no counts round: ONE launch of stores (rotated destination order: at any
// moment the sources write to different receivers) + the data-slot completion flags.
// Work item = one 2 KB part of one chunk (vectors of 16 bytes).
__global__ void __launch_bounds__(512) all_to_all_kernel(CommArgs a, const uint16_t* __restrict__ send, int64_t dst_off,
                                  int64_t chunk_bytes) {
  pdl_wait();
  pdl_trigger();
  a.epoch = load_epoch(a);
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nvec = chunk_bytes / 16;
  const int64_t parts = (nvec + kPartVec - 1) / kPartVec;
  const int64_t n_items = parts * a.ep;
  for (int64_t w = gwarp; w < n_items; w += nwarps) {
    // destination-major with rotation: items [i*parts, (i+1)*parts) go to rank (rank+1+i)%EP
    const int i = static_cast<int>(w / parts);
    const int64_t part = w - static_cast<int64_t>(i) * parts;
    const int q = (a.rank + 1 + i) % a.ep;
    const int64_t v0 = part * kPartVec;
    const int nv = static_cast<int>((nvec - v0) < kPartVec ? (nvec - v0) : kPartVec);
    const uint4* src = reinterpret_cast<const uint4*>(
        reinterpret_cast<const char*>(send) + static_cast<int64_t>(q) * chunk_bytes) + v0;
    uint4* dst = reinterpret_cast<uint4*>(peer_base(a, q) + dst_off +
                                          static_cast<int64_t>(a.rank) * chunk_bytes) + v0;
    copy_part(dst, src, nv, 0, lane);
  }
  signal_done(a, kSlotData, /*wait_after=*/true);
}

// Up to 2 blocks of 512 threads per SM (all co-resident: blocks spin on peer flags), and no
// more than one block per 32 work items (2 KB row parts): small messages are latency-bound,
// and every extra block adds to the launch and to the last-block count.
// With an SM budget (a transfer running beside a GEMM on another stream) every block also
// reserves unused dynamic shared memory, so it cannot be co-scheduled on an SM that holds a
// ~215 KB GEMM CTA: the copy blocks stay on the SMs the GEMM left free instead of stealing
// issue and load/store slots from GEMM CTAs.
int transfer_smem(const CommArgs& a) { return a.blocks > 0 ? 32 * 1024 : 0; }

int transfer_blocks(const CommArgs& a, int64_t rows) {
  int64_t b = a.blocks > 0 ? a.blocks : 2 * num_sms();
  const int64_t parts = (a.d / 8 + 127) / 128;
  const int64_t need = (rows * parts + 31) / 32;
  if (need < b) b = need;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

#ifdef MOE_TRACE
extern "C" int moe_debug_trace(unsigned long long* out) {   // [64][8]
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)));
}
#endif

cudaError_t launch_wait_flags(const CommArgs& a, int slot, cudaStream_t s) {
  launch_k(wait_flags_kernel, dim3(1), dim3(32), 0, s, a, slot);
  return cudaGetLastError();
}

cudaError_t launch_dispatch(const CommArgs& a, const int32_t* counts, int32_t* layout,
                            int64_t recv_rows_cap, const uint16_t* src, int64_t dst_off,
                            uint16_t* local_dst, int s0, int s1, cudaStream_t s) {
  const int64_t rows = a.T * a.k * (s1 - s0) / a.E_l + a.T;   // range share (+ slack)
  launch_k(forward_transfer_kernel<0>, dim3(transfer_blocks(a, rows)), dim3(512), transfer_smem(a),
      s, a, layout, counts, recv_rows_cap, src, dst_off, local_dst, nullptr, nullptr, nullptr,
      nullptr, nullptr, s0, s1);
  return cudaGetLastError();
}

cudaError_t launch_combine_bwd_transfer(const CommArgs& a, int32_t* layout, int64_t dst_off,
                                        uint16_t* local_dst, const int32_t* dest_row,
                                        const float* gates, const uint16_t* dy, const uint16_t* ys,
                                        float* dgates, int s0, int s1, cudaStream_t s) {
  launch_k(forward_transfer_kernel<1>, dim3(transfer_blocks(a, a.T * a.k)), dim3(512),
      transfer_smem(a), s, a, layout, nullptr, 0, nullptr, dst_off, local_dst, dest_row, gates, dy,
      ys, dgates, s0, s1);
  return cudaGetLastError();
}

cudaError_t launch_reverse_transfer(const CommArgs& a, const int32_t* layout, const uint16_t* src,
                                    int64_t dst_off, cudaStream_t s) {
  // receive rows <= EP * T * k
  launch_k(reverse_transfer_kernel, dim3(transfer_blocks(a, a.T * a.k * a.ep)), dim3(512),
      transfer_smem(a), s, a, layout, src, dst_off);
  return cudaGetLastError();
}

cudaError_t launch_all_to_all(const CommArgs& a, const void* send, int64_t dst_off,
                              int64_t chunk_bytes, cudaStream_t s) {
  const int64_t items = a.ep * ((chunk_bytes / 16 + kPartVec - 1) / kPartVec);
  int64_t b = a.blocks > 0 ? a.blocks : 2 * num_sms();
  const int64_t need = (items + 15) / 16;     // 16 warps per block, one 2 KB part each
  if (need < b) b = need;
  launch_k(all_to_all_kernel, dim3(static_cast<unsigned>(b < 1 ? 1 : b)), dim3(512), 0, s, a,
           static_cast<const uint16_t*>(send), dst_off, chunk_bytes);
  return cudaGetLastError();
}

cudaError_t launch_migrate(const CommArgs& a, const MigrateList& ml, const void* src,
                           int64_t dst_off, int64_t bytes_per_expert, cudaStream_t s) {
  const int64_t rows = static_cast<int64_t>(ml.n) * ((bytes_per_expert / 16 + kMigRowVec - 1) / kMigRowVec);
  int64_t b = a.blocks > 0 ? a.blocks : 2 * num_sms();
  const int64_t need = (rows + 31) / 32;
  if (need < b) b = need;
  launch_k(migrate_kernel, dim3(static_cast<unsigned>(b < 1 ? 1 : b)), dim3(512), 0, s, a, ml,
           static_cast<const uint16_t*>(src), dst_off, bytes_per_expert);
  return cudaGetLastError();
}

cudaError_t launch_dedup_forward(const CommArgs& a, int mode, int32_t* layout, int32_t* dlayout,
                                 const int32_t* counts, const int32_t* ntok,
                                 int64_t recv_rows_cap, const uint16_t* src,
                                 const int32_t* pdest, const int32_t* dest_row,
                                 const int32_t* topk_idx, const float* gates, int64_t tok_off,
                                 int64_t rlist_off, int64_t glist_off, const uint16_t* ys,
                                 float* dgates, cudaStream_t s) {
  const int64_t rows = a.T * (a.k < a.ep ? a.k : a.ep) + (ys ? a.T * a.k : 0);   // work bound
  if (mode == 0)
    launch_k(dedup_forward_kernel<0>, dim3(transfer_blocks(a, rows)), dim3(512), transfer_smem(a), s,
        a, layout, dlayout, counts, ntok, recv_rows_cap, src, pdest, dest_row, topk_idx, gates,
        tok_off, rlist_off, glist_off, ys, dgates);
  else
    launch_k(dedup_forward_kernel<1>, dim3(transfer_blocks(a, rows)), dim3(512), transfer_smem(a), s,
        a, layout, dlayout, counts, ntok, recv_rows_cap, src, pdest, dest_row, topk_idx, gates,
        tok_off, rlist_off, glist_off, ys, dgates);
  return cudaGetLastError();
}

cudaError_t launch_dedup_expand(const CommArgs& a, int mode, const int32_t* layout,
                                const int32_t* dlayout, const uint16_t* tok,
                                const int32_t* rlist, const float* glist, const uint16_t* O,
                                uint16_t* dst, float* dg_own, cudaStream_t s) {
  // local kernel, sized like the transfer it follows (an SM budget beside a GEMM applies too)
  const int64_t rows = a.T * a.k * a.ep;   // receive rows bound
  if (mode == 0)
    launch_k(dedup_expand_kernel<0>, dim3(transfer_blocks(a, rows)), dim3(512), transfer_smem(a), s,
        a, layout, dlayout, tok, rlist, glist, O, dst, dg_own);
  else
    launch_k(dedup_expand_kernel<1>, dim3(transfer_blocks(a, rows)), dim3(512), transfer_smem(a), s,
        a, layout, dlayout, tok, rlist, glist, O, dst, dg_own);
  return cudaGetLastError();
}

cudaError_t launch_dedup_reduce(const CommArgs& a, int mode, const int32_t* dlayout,
                                const int32_t* rlist, const float* glist, const uint16_t* rows,
                                const float* dg_own, int64_t part_off, int64_t dgpart_off,
                                cudaStream_t s) {
  const int64_t n = a.T * a.ep;   // pairs received bound
  if (mode == 0)
    launch_k(dedup_reduce_kernel<0>, dim3(transfer_blocks(a, n)), dim3(512), transfer_smem(a), s, a,
        dlayout, rlist, glist, rows, dg_own, part_off, dgpart_off);
  else
    launch_k(dedup_reduce_kernel<1>, dim3(transfer_blocks(a, n)), dim3(512), transfer_smem(a), s, a,
        dlayout, rlist, glist, rows, dg_own, part_off, dgpart_off);
  return cudaGetLastError();
}

}  // namespace moe
