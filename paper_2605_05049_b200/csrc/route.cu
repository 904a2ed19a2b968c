// route.cu -- F1 top-k gating, B1 route_bwd and B0 router backward (SIMT, fp32).
//
// PAPER.md:50-51, 110-111, 121 (learned top-k gating); readings R1-R3:
// select on the fp32 logits, descending value, ties to the lower expert index,
// -0.0 == +0.0, NaN below -inf; gates = softmax over the k selected logits (k>1),
// full-softmax probability of the top expert (k=1).
#include "common.cuh"
#include "internal.h"

namespace moe {
namespace {

constexpr int kMaxE = 1024;               // experts per token handled by one warp
constexpr int kPerLane = kMaxE / 32;

// Order-preserving 32-bit key of an fp32 logit: larger value -> larger key;
// -0.0 and +0.0 map to the same key; NaN maps to 0 (below -inf).
__device__ __forceinline__ uint32_t orderable(float v) {
  if (v != v) return 0u;
  if (v == 0.0f) v = 0.0f;
  uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

template <int PER_LANE>
__global__ void route_kernel(const float* __restrict__ logits, int64_t T, int E, int k,
                             int32_t* __restrict__ topk_idx, float* __restrict__ gates) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const float* row = logits + t * E;
  float v[PER_LANE];
  uint64_t key[PER_LANE];
#pragma unroll
  for (int i = 0; i < PER_LANE; ++i) {
    const int e = i * 32 + lane;  // coalesced: consecutive lanes read consecutive experts
    v[i] = (e < E) ? row[e] : 0.f;
    key[i] = (e < E) ? ((static_cast<uint64_t>(orderable(v[i])) << 32) | (0xFFFFFFFFu - e)) : 0ull;
  }
  float sel0 = 0.f;
  float mine = 0.f;  // lane j keeps the j-th selected logit (k <= 32)
  for (int j = 0; j < k; ++j) {
    uint64_t best = 0ull;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i) best = key[i] > best ? key[i] : best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    const int e = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFull));
    // owner lane clears the winner and broadcasts its value
    float val = 0.f;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i)
      if (i * 32 + lane == e) { key[i] = 0ull; val = v[i]; }
    val = __shfl_sync(0xffffffffu, val, e & 31);
    if (j == 0) sel0 = val;
    if (lane == j) mine = val;
    if (lane == 0) topk_idx[t * k + j] = e;
  }
  if (k == 1) {
    // full softmax probability of the top expert: 1 / sum_e exp(l_e - l_0)
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER_LANE; ++i)
      if (i * 32 + lane < E) s += expf(v[i] - sel0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) gates[t] = 1.f / s;
  } else {
    const float z = (lane < k) ? expf(mine - sel0) : 0.f;
    float denom = z;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
    if (lane < k) gates[t * k + lane] = z / denom;
  }
}

// B1: dl[t, e_j] = g_j (dg_j - sum_i g_i dg_i); k = 1: dl_e = dg g0 (delta - p_e).
__global__ void route_bwd_kernel(const float* __restrict__ logits, const int32_t* __restrict__ idx,
                                 const float* __restrict__ gates, const float* __restrict__ dgates,
                                 int64_t T, int E, int k, float* __restrict__ dl) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  float g = 0.f, dg = 0.f;
  int e_sel = -1;
  if (lane < k) {
    g = gates[t * k + lane];
    dg = dgates[t * k + lane];
    e_sel = idx[t * k + lane];
  }
  float s = g * dg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (k == 1) {
    const float g0 = __shfl_sync(0xffffffffu, g, 0);
    const float dg0 = __shfl_sync(0xffffffffu, dg, 0);
    const int e0 = __shfl_sync(0xffffffffu, e_sel, 0);
    const float* row = logits + t * E;
    float mx = -INFINITY;
    for (int e = lane; e < E; e += 32) mx = fmaxf(mx, row[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float z = 0.f;
    for (int e = lane; e < E; e += 32) z += expf(row[e] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    for (int e = lane; e < E; e += 32) {
      const float pe = expf(row[e] - mx) / z;
      dl[t * E + e] = dg0 * g0 * ((e == e0 ? 1.f : 0.f) - pe);
    }
    return;
  }
  const float val = g * (dg - s);
  for (int e = lane; e < E; e += 32) {
    float out = 0.f;
    for (int j = 0; j < k; ++j) {
      const int ej = __shfl_sync(0xffffffffu, e_sel, j);
      const float vj = __shfl_sync(0xffffffffu, val, j);
      if (ej == e) out = vj;
    }
    dl[t * E + e] = out;
  }
}

// B0 (part 1): dx_router[t, c] = sum_e dl[t,e] w_r[e,c].  Block: 32 tokens x 256 columns;
// dl tile staged transposed in smem ([e][t]) so every column thread reads broadcasts.
template <int TT>
__global__ void router_dx_kernel(const uint16_t* __restrict__ w_r, const float* __restrict__ dl,
                                 int64_t T, int d, int E, float* __restrict__ dx) {
  extern __shared__ float s_dl[];  // [E][TT]
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * TT;
  for (int i = threadIdx.x; i < TT * E; i += blockDim.x) {
    const int tt = i / E, e = i % E;
    s_dl[e * TT + tt] = (t0 + tt < T) ? dl[(t0 + tt) * E + e] : 0.f;
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float acc[TT];
#pragma unroll
  for (int i = 0; i < TT; ++i) acc[i] = 0.f;
  for (int e = 0; e < E; ++e) {
    const float w = __uint_as_float(static_cast<uint32_t>(w_r[static_cast<int64_t>(e) * d + c]) << 16);
    const float4* srow = reinterpret_cast<const float4*>(s_dl + e * TT);
#pragma unroll
    for (int i = 0; i < TT / 4; ++i) {
      const float4 v = srow[i];
      acc[4 * i] += v.x * w; acc[4 * i + 1] += v.y * w;
      acc[4 * i + 2] += v.z * w; acc[4 * i + 3] += v.w * w;
    }
  }
#pragma unroll
  for (int i = 0; i < TT; ++i)
    if (t0 + i < T) dx[(t0 + i) * d + c] = acc[i];
}

// B0 (part 2): dw_r[e, c] (+)= sum_t dl[t,e] x[t,c].  Block: ET experts x 256 columns,
// looping over all tokens in a fixed order (deterministic).
template <int ET>
__global__ void router_dw_kernel(const uint16_t* __restrict__ x, const float* __restrict__ dl,
                                 int64_t T, int d, int E, float* __restrict__ dw, int accumulate) {
  constexpr int TCH = 64;
  __shared__ __align__(16) float s_dl[TCH][ET];
  const int e0 = blockIdx.y * ET;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  float acc[ET];
#pragma unroll
  for (int i = 0; i < ET; ++i) acc[i] = 0.f;
  for (int64_t tb = 0; tb < T; tb += TCH) {
    __syncthreads();
    for (int i = threadIdx.x; i < TCH * ET; i += blockDim.x) {
      const int tt = i / ET, e = i % ET;
      s_dl[tt][e] = (tb + tt < T && e0 + e < E) ? dl[(tb + tt) * E + e0 + e] : 0.f;
    }
    __syncthreads();
    if (c < d) {
      const int n = (T - tb < TCH) ? static_cast<int>(T - tb) : TCH;
      for (int tt = 0; tt < n; ++tt) {
        const float xv = __uint_as_float(static_cast<uint32_t>(x[(tb + tt) * d + c]) << 16);
        const float4* srow = reinterpret_cast<const float4*>(&s_dl[tt][0]);
#pragma unroll
        for (int i = 0; i < ET / 4; ++i) {
          const float4 v = srow[i];
          acc[4 * i] += v.x * xv; acc[4 * i + 1] += v.y * xv;
          acc[4 * i + 2] += v.z * xv; acc[4 * i + 3] += v.w * xv;
        }
      }
    }
  }
  if (c >= d) return;
#pragma unroll
  for (int i = 0; i < ET; ++i) {
    if (e0 + i < E) {
      float* p = dw + static_cast<int64_t>(e0 + i) * d + c;
      *p = accumulate ? (*p + acc[i]) : acc[i];
    }
  }
}

}  // namespace

cudaError_t launch_route(const float* logits, int64_t T, int E, int k, int32_t* topk_idx,
                         float* gates, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (T * 32 + threads - 1) / threads;
  if (E <= 32) route_kernel<1><<<blocks, threads, 0, s>>>(logits, T, E, k, topk_idx, gates);
  else if (E <= 64) route_kernel<2><<<blocks, threads, 0, s>>>(logits, T, E, k, topk_idx, gates);
  else if (E <= 128) route_kernel<4><<<blocks, threads, 0, s>>>(logits, T, E, k, topk_idx, gates);
  else if (E <= 256) route_kernel<8><<<blocks, threads, 0, s>>>(logits, T, E, k, topk_idx, gates);
  else route_kernel<kPerLane><<<blocks, threads, 0, s>>>(logits, T, E, k, topk_idx, gates);
  return cudaGetLastError();
}

cudaError_t launch_route_bwd(const float* logits, const int32_t* topk_idx, const float* gates,
                             const float* dgates, int64_t T, int E, int k, float* dlogits,
                             cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (T * 32 + threads - 1) / threads;
  route_bwd_kernel<<<blocks, threads, 0, s>>>(logits, topk_idx, gates, dgates, T, E, k, dlogits);
  return cudaGetLastError();
}

cudaError_t launch_router_bwd(const uint16_t* x, const uint16_t* w_r, const float* dlogits,
                              int64_t T, int d, int E, float* dx_router, float* dw_r,
                              int accumulate, cudaStream_t s) {
  if (T > 0 && dx_router) {
    constexpr int TT = 32;
    dim3 grid((d + 255) / 256, static_cast<unsigned>((T + TT - 1) / TT));
    size_t smem = static_cast<size_t>(TT) * E * sizeof(float);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(router_dx_kernel<TT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    router_dx_kernel<TT><<<grid, 256, smem, s>>>(w_r, dlogits, T, d, E, dx_router);
  }
  if (dw_r) {
    if (E <= 8) {
      dim3 grid((d + 255) / 256, 1);
      router_dw_kernel<8><<<grid, 256, 0, s>>>(x, dlogits, T, d, E, dw_r, accumulate);
    } else {
      dim3 grid((d + 255) / 256, (E + 31) / 32);
      router_dw_kernel<32><<<grid, 256, 0, s>>>(x, dlogits, T, d, E, dw_r, accumulate);
    }
  }
  return cudaGetLastError();
}

}  // namespace moe
