// permute.cu -- F2 permute (histogram, scan, capacity, scatter), B2 permute_bwd,
// F6 gate-weighted unpermute.  HBM-bound row movement with 16-byte vectors.
//
// Positions are deterministic and bit-exact (no atomic ordering): assignments are
// visited in slot-major order a = j*T + t (reading R5, PAPER.md:129 token dropping),
// the rank of an assignment among equal experts is
//   (earlier chunks, scanned)  +  (earlier warps of the chunk, scanned)  +
//   (earlier lanes of the warp, __match_any_sync + popc)
// and C = ceil(cf*k*T/E) decides kept/dropped (reading R4).
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int kChunk = 1024;  // assignments per block in passes 1 and 3 (32 warps x 32)

__device__ __forceinline__ int expert_of(const int32_t* idx, int64_t a, int64_t T, int k) {
  const int64_t t = a % T, j = a / T;
  return idx[t * k + j];
}

// Pass 1: per-chunk expert histogram; the last block to finish (ticket) then runs pass 2:
// per-expert exclusive scan over chunks (in place -> chunk base), capacity clamp, counts and
// off = exclusive scan of counts.  One launch instead of two.
// With `layout` (the EP = 1 local path, moe_permute_dispatch_local) the last block also writes
// the layout record moe_dispatch would write -- counts_all (= counts), the rows and the
// 128-aligned segment base of every local slot (expert_at[slot] = expert) -- and
// shift[e] = seg_base[slot of e] - off[e], the send-row -> receive-row offset of expert e.
__global__ void hist_scan_kernel(const int32_t* __restrict__ idx, int64_t T, int k, int E,
                                 int64_t C, int32_t* __restrict__ chunk_hist /*[nchunks][E]*/,
                                 int32_t* __restrict__ counts, int32_t* __restrict__ off,
                                 int32_t* __restrict__ ticket, int32_t* __restrict__ layout,
                                 const int32_t* __restrict__ expert_at,
                                 int32_t* __restrict__ shift) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int32_t s_hist[];   // [E]
  __shared__ int s_last;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  __syncthreads();
  const int64_t a = static_cast<int64_t>(blockIdx.x) * kChunk + threadIdx.x;
  if (a < T * k) atomicAdd(&s_hist[expert_of(idx, a, T, k)], 1);  // order-free count
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_hist[static_cast<int64_t>(blockIdx.x) * E + e] = s_hist[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nchunks = gridDim.x;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    int c = 0;
    for (; c + 8 <= nchunks; c += 8) {   // 8 independent loads in flight
      int32_t h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = __ldcg(chunk_hist + static_cast<int64_t>(c + q) * E + e);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        chunk_hist[static_cast<int64_t>(c + q) * E + e] = run;
        run += h[q];
      }
    }
    for (; c < nchunks; ++c) {
      const int32_t h = __ldcg(chunk_hist + static_cast<int64_t>(c) * E + e);
      chunk_hist[static_cast<int64_t>(c) * E + e] = run;
      run += h;
    }
    const int32_t kept = (C >= 0 && run > C) ? static_cast<int32_t>(C) : run;
    counts[e] = kept;
    s_hist[e] = kept;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = run;
      run += s_hist[e];
    }
    off[E] = run;
    *ticket = 0;   // for the next call (stream-ordered)
    if (layout) {
      int32_t seg = 0;
      for (int sl = 0; sl < E; ++sl) {
        const int e = expert_at[sl];
        const int32_t rows = s_hist[e];
        layout[e] = rows;                       // counts_all[0][e]
        layout[E + sl] = rows;                  // expert_rows[slot]
        layout[2 * E + sl] = seg;               // seg_base[slot]
        shift[e] = seg - off[e];
        seg += (rows + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
      }
      layout[3 * E] = seg;
    }
  }
}

// Pass 2: stable rank inside the chunk -> p, kept, dest_row.
__global__ void rank_kernel(const int32_t* __restrict__ idx, int64_t T, int k, int E, int64_t C,
                            const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ off,
                            int32_t* __restrict__ dest_row, int32_t* __restrict__ slot_of_row) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int32_t s_wcnt[];  // [32 warps][E]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) s_wcnt[i] = 0;
  __syncthreads();
  const int64_t a = static_cast<int64_t>(blockIdx.x) * kChunk + threadIdx.x;
  const bool live = a < T * k;
  const int e = live ? expert_of(idx, a, T, k) : -1 - lane;  // unique dummies never match
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int in_warp = __popc(peers & ((1u << lane) - 1u));
  if (live && in_warp == 0) s_wcnt[warp * E + e] = __popc(peers);
  __syncthreads();
  for (int ee = threadIdx.x; ee < E; ee += blockDim.x) {  // exclusive scan over warps
    int32_t run = 0;
    for (int w = 0; w < 32; ++w) {
      const int32_t v = s_wcnt[w * E + ee];
      s_wcnt[w * E + ee] = run;
      run += v;
    }
  }
  __syncthreads();
  if (!live) return;
  const int64_t p = static_cast<int64_t>(chunk_base[static_cast<int64_t>(blockIdx.x) * E + e]) +
                    s_wcnt[warp * E + e] + in_warp;
  const bool kept = (C < 0) || (p < C);
  const int64_t t = a % T, j = a / T;
  dest_row[t * k + j] = kept ? static_cast<int32_t>(off[e] + p) : -1;
  // inverse map (send-layout row -> slot t*k+j) for the row-ordered combine_bwd fused into
  // dgrad-1 (moe_combine_bwd_expert_ffn_dh)
  if (kept && slot_of_row) slot_of_row[off[e] + p] = static_cast<int32_t>(t * k + j);
}

// Pass 3: warp per token; read x_t once (4 x 16 B in flight per lane), write each kept row.
// KMAX >= k is a compile-time bound, so the row list lives in registers (static indices).
// With shift (EP = 1 local path) row dest_row + shift[e] of the 128-aligned receive layout is
// written instead, and warps past the tokens zero the padding rows of every segment.
template <int KMAX>
__global__ void scatter_kernel(const uint16_t* __restrict__ x, int32_t* __restrict__ dest_row,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ shift,
                               const int32_t* __restrict__ layout, int64_t T, int d, int k, int E,
                               uint16_t* __restrict__ xs) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int nvec = d / 8;  // 16-byte vectors per row
  if (t >= T) {
    if (!shift) return;
    // padding rows: warp (t - T) zeroes padding row number (t - T) of the whole buffer
    const int64_t pr = t - T;
    int64_t base = 0;
    for (int sl = 0; sl < E; ++sl) {
      const int32_t rows = layout[E + sl], seg = layout[2 * E + sl];
      const int32_t pad = layout[2 * E + sl + 1] - seg - rows;
      if (pr < base + pad) {
        uint4* z = reinterpret_cast<uint4*>(xs + (static_cast<int64_t>(seg) + rows + (pr - base)) * d);
        for (int v = lane; v < nvec; v += 32) z[v] = make_uint4(0u, 0u, 0u, 0u);
        return;
      }
      base += pad;
    }
    return;
  }
  int32_t rows[KMAX];
  bool any = false;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    int32_t r = j < k ? dest_row[t * k + j] : -1;
    if (shift && r >= 0) r += shift[idx[t * k + j]];
    rows[j] = r;
    any |= r >= 0;
  }
  // local mode: dest_row becomes the receive-layout row (where the row was written), so the
  // unpermute / permute_bwd gathers read the GEMM outputs in place (no send-layout copies)
  if (shift && lane == 0) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k) dest_row[t * k + j] = rows[j];
  }
  __syncwarp();
  if (!any) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
  for (int v0 = lane; v0 < nvec; v0 += 128) {   // 4 loads in flight per lane
    uint4 val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + 32 * u < nvec) val[u] = ld_nc_v4(src + v0 + 32 * u);
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (rows[j] < 0) continue;
      uint4* dst = reinterpret_cast<uint4*>(xs + static_cast<int64_t>(rows[j]) * d);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + 32 * u < nvec) dst[v0 + 32 * u] = val[u];
    }
  }
}

// B6 at EP = 1, local (the permute wrote the receive rows into dest_row): for each kept slot
// dO[dest_row] = bf16(g * dy[t]) and dgates = <dy[t], O[dest_row]>, dy read once per token
// for all its slots; the padding rows of dO's segments are zeroed by the warps past the tokens.
// The dot product visits a lane's vectors in increasing v and reduces over the warp as the
// transfer kernel's combine_bwd does, so both paths give identical dgates.
template <int KMAX>
__global__ void combine_bwd_local_kernel(const uint16_t* __restrict__ dy,
                                         const float* __restrict__ gates,
                                         const int32_t* __restrict__ dest_row,
                                         const uint16_t* __restrict__ O,
                                         const int32_t* __restrict__ layout, int64_t T, int d,
                                         int k, int E, float* __restrict__ dgates,
                                         uint16_t* __restrict__ dout) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int nvec = d / 8;
  if (t >= T) {   // padding rows of the receive segments (layout record: expert_rows, seg_base)
    const int64_t pr = t - T;
    int64_t base = 0;
    for (int sl = 0; sl < E; ++sl) {
      const int32_t rows = layout[E + sl], seg = layout[2 * E + sl];
      const int32_t pad = layout[2 * E + sl + 1] - seg - rows;
      if (pr < base + pad) {
        uint4* z = reinterpret_cast<uint4*>(dout + (static_cast<int64_t>(seg) + rows + (pr - base)) * d);
        for (int v = lane; v < nvec; v += 32) z[v] = make_uint4(0u, 0u, 0u, 0u);
        return;
      }
      base += pad;
    }
    return;
  }
  int32_t rw[KMAX];
  float g[KMAX], dot[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    rw[j] = j < k ? dest_row[t * k + j] : -1;
    g[j] = rw[j] >= 0 ? gates[t * k + j] : 0.f;
    dot[j] = 0.f;
  }
  const uint4* pdy = reinterpret_cast<const uint4*>(dy + t * d);
  for (int v0 = lane; v0 < nvec; v0 += 128) {
    uint4 av[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + 32 * u < nvec) av[u] = ld_nc_v4(pdy + v0 + 32 * u);
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (rw[j] < 0) continue;
      const uint4* po = reinterpret_cast<const uint4*>(O + static_cast<int64_t>(rw[j]) * d);
      uint4* pd = reinterpret_cast<uint4*>(dout + static_cast<int64_t>(rw[j]) * d);
      uint4 bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + 32 * u < nvec) bv[u] = ld_nc_v4(po + v0 + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (v0 + 32 * u >= nvec) break;
        pd[v0 + 32 * u] = combine_bwd_vec(av[u], bv[u], g[j], dot[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    if (j >= k) break;
    float v = dot[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) dgates[t * k + j] = rw[j] >= 0 ? v : 0.f;
  }
}

// y[t] = bf16( sum_{j kept} g_{t,j} rows[dest_row[t,j]] (j order) + extra_f32[t] + extra_bf16[t] )
// One warp per token.  KMAX >= k is a compile-time bound so the row list stays in registers
// (static indices, dropped slots skipped in place: the same j-order sum as a compacted list).
template <bool GATED, int KMAX>
__global__ void gather_sum_kernel(const uint16_t* __restrict__ rows, const float* __restrict__ gates,
                                  const int32_t* __restrict__ dest_row, const float* __restrict__ extra_f32,
                                  const uint16_t* __restrict__ extra_bf16, int64_t T, int d, int k,
                                  uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  int32_t rws[KMAX];
  float gs[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    rws[j] = j < k ? dest_row[t * k + j] : -1;
    gs[j] = (GATED && rws[j] >= 0) ? gates[t * k + j] : 1.f;
  }
  const int nvec = d / 8;
  constexpr int kUnroll = KMAX <= 4 ? 2 : 1;   // keep the live row vectors near 8 per lane
#pragma unroll kUnroll
  for (int v = lane; v < nvec; v += 32) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint4 val[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (rws[j] >= 0) val[j] = ld_nc_v4(reinterpret_cast<const uint4*>(rows + static_cast<int64_t>(rws[j]) * d) + v);
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (rws[j] >= 0) acc_bf16x8(acc, val[j], gs[j]);
    if (extra_f32) {
      const float4* pe = reinterpret_cast<const float4*>(extra_f32 + t * d) + 2 * v;
      const float4 a = pe[0], b = pe[1];
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
    }
    if (extra_bf16)
      acc_bf16x8(acc, ld_nc_v4(reinterpret_cast<const uint4*>(extra_bf16 + t * d) + v), 1.f);
    reinterpret_cast<uint4*>(out + t * d)[v] =
        make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]), pack_bf16(acc[4], acc[5]),
                   pack_bf16(acc[6], acc[7]));
  }
}

// B2 + B0 (dgrad part) fused, k > 1: the router gradient dl[t,:] is zero outside the k
// selected experts (softmax over the selected logits, reading R1), so
//   dx[t] = bf16( sum_{j kept} dxs[dest_row[t,j]] + sum_j dl[t,e_j] w_r[e_j,:] + extra[t] )
// in fp32 with a fixed order -- the dense [T,d] fp32 dx_router never touches HBM.
template <int KMAX, int KRMAX>
// minimum resident blocks: k <= 2 keeps 4 (32 warps; 3 measured 25 % slower on Mixtral),
// k = 3..8 two (the one-round-trip iteration needs up to 128 registers)
__global__ void __launch_bounds__(256, KMAX == 2 ? 4 : (KMAX <= 8 ? 2 : 1))
    gather_sum_router_kernel(const uint16_t* __restrict__ dxs,
                                         const int32_t* __restrict__ dest_row,
                                         const int32_t* __restrict__ topk_idx,
                                         const float* __restrict__ dlogits,
                                         const uint16_t* __restrict__ w_r,
                                         const uint16_t* __restrict__ extra_bf16, int64_t T, int d,
                                         int E, int k, int kr, uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  int32_t rws[KRMAX], es[KMAX];
  float dl[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    es[j] = j < k ? topk_idx[t * k + j] : -1;
    dl[j] = es[j] >= 0 ? dlogits[t * E + es[j]] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < KRMAX; ++j)   // row list: dest_row [T,k] (kr = k) or dedup pdest [T,EP]
    rws[j] = j < kr ? dest_row[t * kr + j] : -1;
  const int nvec = d / 8;
  constexpr int kUnroll = KRMAX <= 4 ? 2 : 1;
#pragma unroll kUnroll
  for (int v = lane; v < nvec; v += 32) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    // every load of the iteration (the dX rows, the W_r rows, the extra row) is issued before
    // the first use: one memory round trip per iteration instead of two (the summation order
    // is unchanged)
    // (k = 3..8; k <= 2 keeps the two-phase order, measured 20 % faster there: Mixtral 53 vs
    // 64 us, and the k <= 32 instance would spill; DS-MoE k = 6: 149-154 vs 244-247 us)
    uint4 val[KRMAX];
#pragma unroll
    for (int j = 0; j < KRMAX; ++j)
      if (rws[j] >= 0) val[j] = ld_nc_v4(reinterpret_cast<const uint4*>(dxs + static_cast<int64_t>(rws[j]) * d) + v);
    if constexpr (KMAX >= 4 && KMAX <= 8) {
      uint4 wv[KMAX], ev = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (es[j] >= 0) wv[j] = ld_nc_v4(reinterpret_cast<const uint4*>(w_r + static_cast<int64_t>(es[j]) * d) + v);
      if (extra_bf16) ev = ld_nc_v4(reinterpret_cast<const uint4*>(extra_bf16 + t * d) + v);
#pragma unroll
      for (int j = 0; j < KRMAX; ++j)
        if (rws[j] >= 0) acc_bf16x8(acc, val[j], 1.f);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (es[j] >= 0) acc_bf16x8(acc, wv[j], dl[j]);
      if (extra_bf16) acc_bf16x8(acc, ev, 1.f);
    } else {
#pragma unroll
      for (int j = 0; j < KRMAX; ++j)
        if (rws[j] >= 0) acc_bf16x8(acc, val[j], 1.f);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (es[j] >= 0)
          acc_bf16x8(acc, ld_nc_v4(reinterpret_cast<const uint4*>(w_r + static_cast<int64_t>(es[j]) * d) + v),
                     dl[j]);
      if (extra_bf16)
        acc_bf16x8(acc, ld_nc_v4(reinterpret_cast<const uint4*>(extra_bf16 + t * d) + v), 1.f);
    }
    reinterpret_cast<uint4*>(out + t * d)[v] =
        make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]), pack_bf16(acc[4], acc[5]),
                   pack_bf16(acc[6], acc[7]));
  }
}

// dw[e, c] (+)= sum_s part[s][e][c] + part[s][Ep + e][c]  (hi and lo halves), fixed order.
__global__ void sum_partials_kernel(const float* __restrict__ part, int S, int E, int Ep, int d,
                                    float* __restrict__ dw, int accumulate) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(E) * d) return;
  const int64_t e = i / d, c = i % d;
  float s = accumulate ? dw[i] : 0.f;
  for (int p = 0; p < S; ++p) {
    const float* base = part + static_cast<int64_t>(p) * 2 * Ep * d;
    s += base[e * d + c] + base[(Ep + e) * d + c];
  }
  dw[i] = s;
}


// ---------------------------------------------------------------- NEXT-4 dedup pairs
// Reading R18 (oracle/dedup.py `pairs`): token t has a PAIR with owner q iff one of its kept
// slots j has owner(e_j) = place[e_j] / E_l = q.  pdest[t, q] = pair_base[q] + tslot, tslot =
// rank of t among this rank's tokens paired with q (ascending t), pair_base = exclusive scan
// of ntok over q; -1 if no pair.  Two launches over blocks of kPairThreads tokens:
//   mark : owner bitmask per token, per-block pair counts (__syncthreads_count); the last
//          block (ticket) scans the block counts per owner into block bases and ntok
//   write: rank inside the block (warp ballots + warp prefix) + block base -> pdest
constexpr int kPairThreads = 1024;

__global__ void __launch_bounds__(kPairThreads) dedup_mark_kernel(
    const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ dest_row,
    const int32_t* __restrict__ place, int64_t T, int k, int E_l, int EP,
    uint8_t* __restrict__ masks, int32_t* __restrict__ blk /*[nb][EP]: counts -> bases*/,
    int32_t* __restrict__ ntok, int32_t* __restrict__ ticket) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_place[256];
  __shared__ int s_last;
  const int E = E_l * EP;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_place[i] = place[i];
  __syncthreads();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kPairThreads + threadIdx.x;
  uint32_t m = 0;
  if (t < T) {
    for (int j = 0; j < k; ++j)
      if (dest_row[t * k + j] >= 0) m |= 1u << (s_place[topk_idx[t * k + j]] / E_l);
    masks[t] = static_cast<uint8_t>(m);
  }
  for (int q = 0; q < EP; ++q) {
    const int c = __syncthreads_count((m >> q) & 1u);
    if (threadIdx.x == 0) blk[blockIdx.x * EP + q] = c;
  }
  // last block: exclusive scan of the block counts per owner, offset by pair_base[q]
  __threadfence();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int32_t pair_base = 0;
    for (int q = 0; q < EP; ++q) {
      int32_t carry = 0;
      for (int b0 = 0; b0 < static_cast<int>(gridDim.x); b0 += 32) {
        const int b = b0 + lane;
        const int32_t c = b < static_cast<int>(gridDim.x) ? __ldcg(blk + b * EP + q) : 0;
        int32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (b < static_cast<int>(gridDim.x)) blk[b * EP + q] = pair_base + carry + x - c;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) ntok[q] = carry;
      pair_base += carry;
    }
    if (lane == 0) *ticket = 0;   // ready for the next call
  }
}

__global__ void __launch_bounds__(kPairThreads) dedup_pdest_kernel(
    const uint8_t* __restrict__ masks, const int32_t* __restrict__ blk, int64_t T, int EP,
    int32_t* __restrict__ pdest) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t s_warp[kPairThreads / 32][MOE_MAX_EP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kPairThreads + threadIdx.x;
  const uint32_t m = t < T ? masks[t] : 0u;
  int32_t below[MOE_MAX_EP];
#pragma unroll
  for (int q = 0; q < MOE_MAX_EP; ++q) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (m >> q) & 1u);
    below[q] = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[warp][q] = __popc(bal);
  }
  __syncthreads();
  if (threadIdx.x < MOE_MAX_EP) {   // exclusive scan over the block's warps, per owner
    const int q = threadIdx.x;
    int32_t run = 0;
    for (int w = 0; w < kPairThreads / 32; ++w) {
      const int32_t v = s_warp[w][q];
      s_warp[w][q] = run;
      run += v;
    }
  }
  __syncthreads();
  if (t >= T) return;
  for (int q = 0; q < EP; ++q)
    pdest[t * EP + q] = ((m >> q) & 1u) ? blk[blockIdx.x * EP + q] + s_warp[warp][q] + below[q] : -1;
}

// dgates[t,j] = dgpart[pdest[t, owner(e_j)] * k + j] for kept slots, 0 for dropped ones.
__global__ void dedup_dgates_kernel(const int32_t* __restrict__ dest_row,
                                    const int32_t* __restrict__ topk_idx,
                                    const int32_t* __restrict__ pdest,
                                    const int32_t* __restrict__ place, int E_l, int EP,
                                    const float* __restrict__ dgpart, int64_t T, int k,
                                    float* __restrict__ dgates) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= T * k) return;
  const int64_t t = i / k;
  const int j = static_cast<int>(i - t * k);
  float v = 0.f;
  if (dest_row[i] >= 0) {
    const int q = place[topk_idx[i]] / E_l;
    v = dgpart[static_cast<int64_t>(pdest[t * EP + q]) * k + j];
  }
  dgates[i] = v;
}

}  // namespace

cudaError_t launch_permute_bwd_router(const uint16_t* dxs, const int32_t* dest_row,
                                      const int32_t* topk_idx, const float* dlogits,
                                      const uint16_t* w_r, const uint16_t* dx_extra, int64_t T,
                                      int d, int E, int k, uint16_t* dx, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const dim3 grid(static_cast<unsigned>((T * 32 + threads - 1) / threads));
#define MOE_GSR(K_, KR_) launch_k(gather_sum_router_kernel<K_, KR_>, grid, dim3(threads), 0, s, dxs, \
                                  dest_row, topk_idx, dlogits, w_r, dx_extra, T, d, E, k, k, dx)
  if (k <= 2) MOE_GSR(2, 2);
  else if (k <= 4) MOE_GSR(4, 4);
  else if (k <= 8) MOE_GSR(8, 8);
  else MOE_GSR(32, 32);
#undef MOE_GSR
  return cudaGetLastError();
}

cudaError_t launch_permute_bwd_router_rows(const uint16_t* dxs, const int32_t* rows, int kr,
                                           const int32_t* topk_idx, const float* dlogits,
                                           const uint16_t* w_r, const uint16_t* dx_extra,
                                           int64_t T, int d, int E, int k, uint16_t* dx,
                                           cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const dim3 grid(static_cast<unsigned>((T * 32 + threads - 1) / threads));
#define MOE_GSR(K_, KR_) launch_k(gather_sum_router_kernel<K_, KR_>, grid, dim3(threads), 0, s, dxs, \
                                  rows, topk_idx, dlogits, w_r, dx_extra, T, d, E, k, kr, dx)
  if (kr <= 2 && k <= 2) MOE_GSR(2, 2);
  else if (kr <= 4 && k <= 4) MOE_GSR(4, 4);
  else if (kr <= 8 && k <= 8) MOE_GSR(8, 8);
  else MOE_GSR(32, 32);
#undef MOE_GSR
  return cudaGetLastError();
}

int64_t dedup_scratch_ints(int64_t T, int EP) {
  const int64_t nb = (T + kPairThreads - 1) / kPairThreads;
  return (T + 3) / 4 + (nb > 0 ? nb : 1) * EP + 1;   // masks (bytes), block counts, ticket
}

cudaError_t launch_dedup_pairs(const int32_t* topk_idx, const int32_t* dest_row,
                               const int32_t* place, int64_t T, int k, int E_l, int EP,
                               int32_t* pdest, int32_t* ntok, int32_t* scratch, cudaStream_t s) {
  if (T == 0) return cudaMemsetAsync(ntok, 0, sizeof(int32_t) * EP, s);
  const int64_t nb = (T + kPairThreads - 1) / kPairThreads;
  uint8_t* masks = reinterpret_cast<uint8_t*>(scratch);
  int32_t* blk = scratch + (T + 3) / 4;
  int32_t* ticket = blk + nb * EP;
  launch_k(dedup_mark_kernel, dim3(static_cast<unsigned>(nb)), dim3(kPairThreads), 0, s, topk_idx,
      dest_row, place, T, k, E_l, EP, masks, blk, ntok, ticket);
  launch_k(dedup_pdest_kernel, dim3(static_cast<unsigned>(nb)), dim3(kPairThreads), 0, s, masks,
      blk, T, EP, pdest);
  return cudaGetLastError();
}

cudaError_t launch_dedup_dgates(const int32_t* dest_row, const int32_t* topk_idx,
                                const int32_t* pdest, const int32_t* place, int E_l, int EP,
                                const float* dgpart, int64_t T, int k, float* dgates,
                                cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int64_t n = T * k;
  launch_k(dedup_dgates_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s,
      dest_row, topk_idx, pdest, place, E_l, EP, dgpart, T, k, dgates);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(const float* part, int S, int E, int Ep, int d, float* dw,
                                int accumulate, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(E) * d;
  launch_k(sum_partials_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, part,
      S, E, Ep, d, dw, accumulate);
  return cudaGetLastError();
}

int64_t permute_scratch_ints(int64_t T, int k, int E) {
  const int64_t nchunks = (T * k + kChunk - 1) / kChunk;
  // chunk bases, off [E+1], block ticket, shift [E] (EP = 1 local path)
  return (nchunks > 0 ? nchunks : 1) * E + E + 1 + 1 + E;
}

cudaError_t launch_permute(const uint16_t* x, const int32_t* topk_idx, int64_t T, int d, int E,
                           int k, int64_t C, int32_t* counts, int32_t* dest_row, uint16_t* xs,
                           int32_t* scratch, cudaStream_t s, int32_t* layout,
                           const int32_t* expert_at, int64_t pad_rows_max, int32_t* slot_of_row) {
  const int64_t nA = T * k;
  const int nchunks = static_cast<int>((nA + kChunk - 1) / kChunk);
  int32_t* chunk_hist = scratch;
  int32_t* off = scratch + static_cast<int64_t>(nchunks > 0 ? nchunks : 1) * E;
  int32_t* ticket = off + E + 1;
  int32_t* shift = ticket + 1;
  if (nchunks == 0) {
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s);
    if (layout) cudaMemsetAsync(layout, 0, sizeof(int32_t) * (3 * E + 1), s);
    return cudaGetLastError();
  }
  launch_k(hist_scan_kernel, dim3(nchunks), dim3(kChunk), E * sizeof(int32_t), s, topk_idx, T, k,
           E, C, chunk_hist, counts, off, ticket, layout, expert_at, layout ? shift : nullptr);
  const size_t smem = static_cast<size_t>(32) * E * sizeof(int32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  launch_k(rank_kernel, dim3(nchunks), dim3(kChunk), smem, s, topk_idx, T, k, E, C, chunk_hist, off,
      dest_row, slot_of_row);
  const int threads = 256;
  if (!xs) return cudaGetLastError();   // indices only (the dedup dispatch reads x directly)
  const int64_t warps = T + (layout ? pad_rows_max : 0);
  const dim3 grid(static_cast<unsigned>((warps * 32 + threads - 1) / threads));
  const int32_t* sh = layout ? shift : nullptr;
#define MOE_SC(K_) launch_k(scatter_kernel<K_>, grid, dim3(threads), 0, s, x, dest_row, topk_idx, \
                            sh, layout, T, d, k, E, xs)
  if (k <= 2) MOE_SC(2);
  else if (k <= 4) MOE_SC(4);
  else if (k <= 8) MOE_SC(8);
  else if (k <= 16) MOE_SC(16);
  else MOE_SC(32);
#undef MOE_SC
  return cudaGetLastError();
}

cudaError_t launch_permute_bwd(const uint16_t* dxs, const int32_t* dest_row, const float* dx_acc,
                               const uint16_t* dx_extra, int64_t T, int d, int k, uint16_t* dx,
                               cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const dim3 grid(static_cast<unsigned>((T * 32 + threads - 1) / threads));
#define MOE_GS(K_) launch_k(gather_sum_kernel<false, K_>, grid, dim3(threads), 0, s, dxs, nullptr, \
                            dest_row, dx_acc, dx_extra, T, d, k, dx)
  if (k <= 2) MOE_GS(2);
  else if (k <= 4) MOE_GS(4);
  else if (k <= 8) MOE_GS(8);
  else MOE_GS(32);
#undef MOE_GS
  return cudaGetLastError();
}

cudaError_t launch_combine_bwd_local(const uint16_t* dy, const float* gates,
                                     const int32_t* dest_row, const uint16_t* O,
                                     const int32_t* layout, int64_t T, int d, int k, int E,
                                     int64_t pad_rows_max, float* dgates, uint16_t* dout,
                                     cudaStream_t s) {
  const int threads = 256;
  const int64_t warps = T + pad_rows_max;
  if (warps == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((warps * 32 + threads - 1) / threads));
#define MOE_CB(K_) launch_k(combine_bwd_local_kernel<K_>, grid, dim3(threads), 0, s, dy, gates, \
                            dest_row, O, layout, T, d, k, E, dgates, dout)
  if (k <= 2) MOE_CB(2);
  else if (k <= 4) MOE_CB(4);
  else if (k <= 8) MOE_CB(8);
  else MOE_CB(32);
#undef MOE_CB
  return cudaGetLastError();
}

cudaError_t launch_unpermute(const uint16_t* ys, const float* gates, const int32_t* dest_row,
                             const uint16_t* y_extra, int64_t T, int d, int k, uint16_t* y,
                             cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const dim3 grid(static_cast<unsigned>((T * 32 + threads - 1) / threads));
#define MOE_GS(K_) launch_k(gather_sum_kernel<true, K_>, grid, dim3(threads), 0, s, ys, gates, \
                            dest_row, nullptr, y_extra, T, d, k, y)
  if (k <= 2) MOE_GS(2);
  else if (k <= 4) MOE_GS(4);
  else if (k <= 8) MOE_GS(8);
  else MOE_GS(32);
#undef MOE_GS
  return cudaGetLastError();
}

}  // namespace moe
