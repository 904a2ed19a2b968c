// gemm.cu -- persistent grouped GEMM on the 5th-generation tensor cores (sm_100a).
//
// Serves every dense contraction on the hot path:
//   F0 router logits   x[T,d] . w_r[E,d]^T                       (M-grouped, 1 group)
//   F4 GEMM1           xr_g . w_gu_g^T  -> G,U,H (SwiGLU epilogue)   (M-grouped)
//   F4 GEMM2           H_g  . w_down_g^T -> O                        (M-grouped)
//   B4 dgrad-1         dO_g . w_down_g   -> dH -> dG,dU (dSwiGLU)     (M-grouped, B MN-major)
//   B4 dgrad-2         dGU_g . w_gu_g    -> dX                        (M-grouped, B MN-major)
//   B4 wgrad           dO_g^T H_g, dGU_g^T X_g  (K = the group's rows) (K-grouped, A,B MN-major)
// The paper's expert GEMMs are "tall-and-skinny" per expert;
// here all experts of a rank are ONE persistent launch over a (group, m, n) tile list
// built on the device from the routed row counts, so no host round trip is needed.
//
// Structure (one CTA per SM, 256 threads):
//   warp 0      TMA producer   (cp.async.bulk.tensor, 128B swizzle, mbarrier ring)
//   warp 1      MMA issuer     (tcgen05.mma kind::f16, M=128 x N=BN x K=16, fp32 in TMEM)
//   warp 2      TMEM allocator (2 accumulator stages -> epilogue overlaps the next tile)
//   warps 4..7  epilogue       (tcgen05.ld 32x32b -> fused activation -> global stores)
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace moe {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes = one 128B-swizzle atom row
constexpr int kThreads = 256;
constexpr int kMaxGroups = 256;

struct KParams {
  int M, N, K;
  int n_groups;
  const int32_t* group_rows;
  int64_t rows_cap;
  int64_t b_group_stride, b_split;
  void* out;
  int64_t ld_out;
  const void* aux;
  int64_t ld_aux;
  const float* bias;
  int f;
  int accumulate;
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int ACC_STRIDE = BN < 32 ? 32 : BN;
  static constexpr int TMEM_COLS = (2 * ACC_STRIDE <= 32)    ? 32
                                   : (2 * ACC_STRIDE <= 64)  ? 64
                                   : (2 * ACC_STRIDE <= 128) ? 128
                                   : (2 * ACC_STRIDE <= 256) ? 256
                                                             : 512;
  // ring + barriers/tables + alignment slack
  static constexpr int SMEM = STAGES * STAGE_BYTES + 4096 + 1024;
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Decoded work tile.
struct Tile {
  int g, m, n, nkb;
  int rows_g;   // valid rows of the group
  int seg;      // first row of the group's segment
};

template <bool KGROUPED, int BN>
__device__ __forceinline__ Tile decode_tile(int t, const int* s_tile_prefix, const int* s_seg,
                                            const int* s_rows, int n_groups, const KParams& p) {
  // upper_bound over the tile prefix
  int lo = 0, hi = n_groups;  // find g: prefix[g] <= t < prefix[g+1]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (s_tile_prefix[mid] <= t) lo = mid; else hi = mid;
  }
  Tile tl;
  tl.g = lo;
  tl.rows_g = s_rows[lo];
  tl.seg = s_seg[lo];
  int local = t - s_tile_prefix[lo];
  if (KGROUPED) {
    int mt = ceil_div(p.M, kBM);
    tl.m = local % mt;
    tl.n = local / mt;
    tl.nkb = ceil_div(tl.rows_g, kBK);
  } else {
    int mt = ceil_div(tl.rows_g, kBM);
    tl.m = local % mt;
    tl.n = local / mt;
    tl.nkb = p.K / kBK;
  }
  return tl;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const KParams p) {
  using C = Cfg<BN>;
  constexpr bool KGROUPED = (EPI == kEpiF32Group);
  constexpr uint32_t IDESC = idesc_bf16(kBM, BN, A_MN, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_tile_prefix = reinterpret_cast<int*>(tmem_slot + 4);  // [kMaxGroups+1]
  int* s_seg = s_tile_prefix + kMaxGroups + 1;                   // [kMaxGroups+1]
  int* s_rows = s_seg + kMaxGroups + 1;                          // [kMaxGroups]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_groups = p.n_groups;

  // ---- group tables: seg_base = 128-aligned prefix of rows; tile prefix
  if (warp == 3) {
    const int NT = ceil_div(p.N, BN);
    const int MT = ceil_div(p.M, kBM);
    int seg_carry = 0, tile_carry = 0;
    for (int base = 0; base < n_groups; base += 32) {
      int g = base + lane;
      int rows = (g < n_groups) ? p.group_rows[g] : 0;
      int seg_sz = ((rows + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS) * MOE_ALIGN_ROWS;
      int tiles = (g < n_groups) ? (KGROUPED ? MT * NT : ceil_div(rows, kBM) * NT) : 0;
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
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = s_tile_prefix[n_groups];

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        Tile tl = decode_tile<KGROUPED, BN>(t, s_tile_prefix, s_seg, s_rows, n_groups, p);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          // ---- A
          if (A_MN) {  // K-grouped wgrad: A[m, k] stored [k rows, m cols]
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              tma_load_2d(a_dst + i * 8192, &tmA, &full[stage], tl.m * kBM + i * 64,
                          tl.seg + kb * kBK);
          } else {
            tma_load_2d(a_dst, &tmA, &full[stage], kb * kBK, tl.seg + tl.m * kBM);
          }
          // ---- B
          if (B_MN) {
            const int krow = KGROUPED ? (tl.seg + kb * kBK)
                                      : static_cast<int>(tl.g * p.b_group_stride) + kb * kBK;
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(b_dst + i * 8192, &tmB, &full[stage], tl.n * BN + i * 64, krow);
          } else if (EPI == kEpiSwiGLU) {
            const int r0 = static_cast<int>(tl.g * p.b_group_stride) + tl.n * (BN / 2);
            tma_load_2d(b_dst, &tmB, &full[stage], kb * kBK, r0);
            tma_load_2d(b_dst + (BN / 2) * 128, &tmB, &full[stage], kb * kBK,
                        r0 + static_cast<int>(p.b_split));
          } else {
            tma_load_2d(b_dst, &tmB, &full[stage], kb * kBK,
                        static_cast<int>(tl.g * p.b_group_stride) + tl.n * BN);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        Tile tl = decode_tile<KGROUPED, BN>(t, s_tile_prefix, s_seg, s_rows, n_groups, p);
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
            umma_bf16(d_tmem, adesc, bdesc, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // frees the smem slot when these MMAs complete
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (tl.nkb > 0) umma_commit(&tfull[acc]);
        else mbar_arrive(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // TMEM lane quadrant ew*32 .. ew*32+31
    const int r_in_tile = ew * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      Tile tl = decode_tile<KGROUPED, BN>(t, s_tile_prefix, s_seg, s_rows, n_groups, p);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * C::ACC_STRIDE;
      uint32_t r[32];

      if (EPI == kEpiSwiGLU) {
        const int mi = tl.m * kBM + r_in_tile;
        const int64_t row = static_cast<int64_t>(tl.seg) + mi;
        const bool write = row < p.rows_cap;
        const bool valid = mi < tl.rows_g;
        uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + row * p.ld_out;
#pragma unroll 1
        for (int c0 = 0; c0 < BN / 2; c0 += 32) {
          uint32_t u[32];
          tmem_ld32(tacc + c0, r);
          tmem_ld32(tacc + BN / 2 + c0, u);
          tmem_ld_wait();
          if (write) {
            const int col = tl.n * (BN / 2) + c0;
            uint4* pg = reinterpret_cast<uint4*>(o + col);
            uint4* pu = reinterpret_cast<uint4*>(o + p.f + col);
            uint4* ph = reinterpret_cast<uint4*>(o + 2 * p.f + col);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint32_t gw[4], uw[4], hw[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float g0 = __uint_as_float(r[v * 8 + 2 * q]), g1 = __uint_as_float(r[v * 8 + 2 * q + 1]);
                float u0 = __uint_as_float(u[v * 8 + 2 * q]), u1 = __uint_as_float(u[v * 8 + 2 * q + 1]);
                if (!valid) { g0 = g1 = u0 = u1 = 0.f; }
                // H from the fp32 accumulators (one bf16 rounding of each saved tensor)
                float h0 = g0 / (1.f + __expf(-g0)) * u0;
                float h1 = g1 / (1.f + __expf(-g1)) * u1;
                gw[q] = pack_bf16(g0, g1);
                uw[q] = pack_bf16(u0, u1);
                hw[q] = pack_bf16(h0, h1);
              }
              pg[v] = make_uint4(gw[0], gw[1], gw[2], gw[3]);
              pu[v] = make_uint4(uw[0], uw[1], uw[2], uw[3]);
              ph[v] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            }
          }
        }
      } else if (EPI == kEpiBF16 || EPI == kEpiDSwiGLU) {
        const int mi = tl.m * kBM + r_in_tile;
        const int64_t row = static_cast<int64_t>(tl.seg) + mi;
        const bool write = row < p.rows_cap;
        const bool valid = mi < tl.rows_g;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          tmem_ld32(tacc + c0, r);
          tmem_ld_wait();
          const int col = tl.n * BN + c0;
          if (write && col < p.N) {
            if (EPI == kEpiBF16) {
              uint4* po = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) +
                                                   row * p.ld_out + col);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  w[q] = valid ? pack_bf16(__uint_as_float(r[v * 8 + 2 * q]),
                                           __uint_as_float(r[v * 8 + 2 * q + 1]))
                               : 0u;
                po[v] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            } else {
              // dH -> dG = dH*U*silu'(G), dU = dH*silu(G); G, U from the saved bf16 g_u_h
              const uint16_t* a = reinterpret_cast<const uint16_t*>(p.aux) + row * p.ld_aux;
              const uint4* pg = reinterpret_cast<const uint4*>(a + col);
              const uint4* pu = reinterpret_cast<const uint4*>(a + p.f + col);
              uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + row * p.ld_out;
              uint4* pdg = reinterpret_cast<uint4*>(o + col);
              uint4* pdu = reinterpret_cast<uint4*>(o + p.f + col);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint4 gv = pg[v], uv = pu[v];
                const uint32_t gw_in[4] = {gv.x, gv.y, gv.z, gv.w};
                const uint32_t uw_in[4] = {uv.x, uv.y, uv.z, uv.w};
                uint32_t dgw[4], duw[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float dh0 = __uint_as_float(r[v * 8 + 2 * q]);
                  float dh1 = __uint_as_float(r[v * 8 + 2 * q + 1]);
                  float g0 = bf16_lo(gw_in[q]), g1 = bf16_hi(gw_in[q]);
                  float u0 = bf16_lo(uw_in[q]), u1 = bf16_hi(uw_in[q]);
                  float s0 = 1.f / (1.f + __expf(-g0)), s1 = 1.f / (1.f + __expf(-g1));
                  float dg0 = dh0 * u0 * s0 * (1.f + g0 * (1.f - s0));
                  float dg1 = dh1 * u1 * s1 * (1.f + g1 * (1.f - s1));
                  float du0 = dh0 * g0 * s0, du1 = dh1 * g1 * s1;
                  if (!valid) { dg0 = dg1 = du0 = du1 = 0.f; }
                  dgw[q] = pack_bf16(dg0, dg1);
                  duw[q] = pack_bf16(du0, du1);
                }
                pdg[v] = make_uint4(dgw[0], dgw[1], dgw[2], dgw[3]);
                pdu[v] = make_uint4(duw[0], duw[1], duw[2], duw[3]);
              }
            }
          }
        }
      } else if (EPI == kEpiF32Group) {
        const int row = tl.m * kBM + r_in_tile;
        float* o = reinterpret_cast<float*>(p.out) +
                   static_cast<int64_t>(tl.g) * p.M * p.N + static_cast<int64_t>(row) * p.N;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          if (tl.nkb > 0) {
            tmem_ld32(tacc + c0, r);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) r[q] = 0u;
          }
          const int col = tl.n * BN + c0;
          if (row < p.M && col < p.N) {
            float4* po = reinterpret_cast<float4*>(o + col);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              float4 val = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                       __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
              if (p.accumulate) {
                float4 old = po[v];
                val.x += old.x; val.y += old.y; val.z += old.z; val.w += old.w;
              }
              po[v] = val;
            }
          }
        }
      } else {  // kEpiF32Rows: router logits
        const int64_t row = static_cast<int64_t>(tl.m) * kBM + r_in_tile;
        float* o = reinterpret_cast<float*>(p.out) + row * p.ld_out;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          tmem_ld32(tacc + c0, r);
          tmem_ld_wait();
          if (row < p.rows_cap) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const int col = tl.n * BN + c0 + q;
              if (col < p.N) o[col] = __uint_as_float(r[q]) + (p.bias ? p.bias[col] : 0.f);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
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

bool make_tmap(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
               int box_cols, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn || rows <= 0 || cols <= 0) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch_impl(const GemmProblem& g, cudaStream_t stream) {
  using C = Cfg<BN>;
  CUtensorMap ta, tb;
  // A box: K-major {64 k, 128 rows}; MN-major {64 m, 64 k}
  if (!make_tmap(&ta, g.a_ptr, g.a_rows, g.a_cols, g.a_ld, 64, A_MN ? 64 : kBM))
    return cudaErrorInvalidValue;
  int b_box_rows = B_MN ? 64 : (EPI == kEpiSwiGLU ? BN / 2 : BN);
  if (!make_tmap(&tb, g.b_ptr, g.b_rows, g.b_cols, g.b_ld, 64, b_box_rows))
    return cudaErrorInvalidValue;
  KParams kp;
  kp.M = g.M; kp.N = g.N; kp.K = g.K;
  kp.n_groups = g.n_groups;
  kp.group_rows = g.group_rows;
  kp.rows_cap = g.rows_cap;
  kp.b_group_stride = g.b_group_stride;
  kp.b_split = g.b_split;
  kp.out = g.out; kp.ld_out = g.ld_out;
  kp.aux = g.aux; kp.ld_aux = g.ld_aux;
  kp.bias = g.bias;
  kp.f = g.f;
  kp.accumulate = g.accumulate;
  auto kern = grouped_gemm_kernel<BN, A_MN, B_MN, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<num_sms(), kThreads, C::SMEM, stream>>>(ta, tb, kp);
  return cudaGetLastError();
}

}  // namespace

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_grouped_gemm(const GemmProblem& g, cudaStream_t s) {
  if (g.n_groups <= 0 || g.n_groups > kMaxGroups) return cudaErrorInvalidValue;
  switch (g.epi) {
    case kEpiSwiGLU:
      if (g.BN == 256) return launch_impl<256, false, false, kEpiSwiGLU>(g, s);
      if (g.BN == 128) return launch_impl<128, false, false, kEpiSwiGLU>(g, s);
      break;
    case kEpiBF16:
      if (!g.b_mn) {
        if (g.BN == 256) return launch_impl<256, false, false, kEpiBF16>(g, s);
        if (g.BN == 128) return launch_impl<128, false, false, kEpiBF16>(g, s);
        if (g.BN == 64) return launch_impl<64, false, false, kEpiBF16>(g, s);
      } else {
        if (g.BN == 256) return launch_impl<256, false, true, kEpiBF16>(g, s);
        if (g.BN == 128) return launch_impl<128, false, true, kEpiBF16>(g, s);
        if (g.BN == 64) return launch_impl<64, false, true, kEpiBF16>(g, s);
      }
      break;
    case kEpiDSwiGLU:
      if (g.BN == 256) return launch_impl<256, false, true, kEpiDSwiGLU>(g, s);
      if (g.BN == 128) return launch_impl<128, false, true, kEpiDSwiGLU>(g, s);
      break;
    case kEpiF32Group:
      if (g.BN == 256) return launch_impl<256, true, true, kEpiF32Group>(g, s);
      if (g.BN == 128) return launch_impl<128, true, true, kEpiF32Group>(g, s);
      if (g.BN == 64) return launch_impl<64, true, true, kEpiF32Group>(g, s);
      break;
    case kEpiF32Rows:
      if (g.BN == 256) return launch_impl<256, false, false, kEpiF32Rows>(g, s);
      if (g.BN == 128) return launch_impl<128, false, false, kEpiF32Rows>(g, s);
      if (g.BN == 64) return launch_impl<64, false, false, kEpiF32Rows>(g, s);
      if (g.BN == 16) return launch_impl<16, false, false, kEpiF32Rows>(g, s);
      break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace moe
