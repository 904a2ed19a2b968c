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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

// B0 prologue: split the fp32 router gradient into two bf16 terms, dl = hi + lo + O(2^-16 |dl|),
// laid out [T, 2*Ep] = [hi | lo] (Ep = E rounded up to 8, zero padding, 16-byte rows for TMA):
// read K-major it is the K-concatenation for dl.[W_r; W_r]; read MN-major it is the
// M-stacking for [hi | lo]^T x.  Either way one bf16 tensor-core GEMM gives fp32 accuracy.
__global__ void split_hilo_kernel(const float* __restrict__ dl, int64_t T, int E, int Ep,
                                  uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= T * Ep) return;
  const int64_t t = i / Ep;
  const int e = static_cast<int>(i % Ep);
  const float v = (e < E) ? dl[t * E + e] : 0.f;
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
  out[t * 2 * Ep + e] = *reinterpret_cast<const uint16_t*>(&h);
  out[t * 2 * Ep + Ep + e] = *reinterpret_cast<const uint16_t*>(&l);
}

// [W_r; W_r] stacked at rows 0 and Ep of a [2*Ep, d] buffer (padding rows zero).
__global__ void stack_wr_kernel(const uint16_t* __restrict__ w_r, int E, int Ep, int d,
                                uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(2) * Ep * d) return;
  const int64_t r = i / d, c = i % d;
  const int64_t e = r < Ep ? r : r - Ep;
  out[i] = (e < E) ? w_r[e * d + c] : static_cast<uint16_t>(0);
}

}  // namespace

cudaError_t launch_route(const float* logits, int64_t T, int E, int k, int32_t* topk_idx,
                         float* gates, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (T * 32 + threads - 1) / threads;
  if (E <= 32) launch_k(route_kernel<1>, dim3(blocks), dim3(threads), 0, s, logits, T, E, k, topk_idx, gates);
  else if (E <= 64) launch_k(route_kernel<2>, dim3(blocks), dim3(threads), 0, s, logits, T, E, k, topk_idx, gates);
  else if (E <= 128) launch_k(route_kernel<4>, dim3(blocks), dim3(threads), 0, s, logits, T, E, k, topk_idx, gates);
  else if (E <= 256) launch_k(route_kernel<8>, dim3(blocks), dim3(threads), 0, s, logits, T, E, k, topk_idx, gates);
  else launch_k(route_kernel<kPerLane>, dim3(blocks), dim3(threads), 0, s, logits, T, E, k,
      topk_idx, gates);
  return cudaGetLastError();
}

cudaError_t launch_route_bwd(const float* logits, const int32_t* topk_idx, const float* gates,
                             const float* dgates, int64_t T, int E, int k, float* dlogits,
                             cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (T * 32 + threads - 1) / threads;
  launch_k(route_bwd_kernel, dim3(blocks), dim3(threads), 0, s, logits, topk_idx, gates, dgates, T,
      E, k, dlogits);
  return cudaGetLastError();
}

cudaError_t launch_split_hilo(const float* dl, int64_t T, int E, int Ep, uint16_t* out,
                              cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int64_t n = T * Ep;
  launch_k(split_hilo_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, dl, T,
      E, Ep, out);
  return cudaGetLastError();
}

cudaError_t launch_stack_wr(const uint16_t* w_r, int E, int Ep, int d, uint16_t* out,
                            cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(2) * Ep * d;
  launch_k(stack_wr_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, w_r, E,
      Ep, d, out);
  return cudaGetLastError();
}

}  // namespace moe
