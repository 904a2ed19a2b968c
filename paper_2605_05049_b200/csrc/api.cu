// api.cu -- the C ABI of libmoe (include/moe.h): validation, context, symmetric heap,
// and the launch sequence of every hot-path step.  No compute happens on the host.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.h"

struct moe_ctx {
  moe_shape s;
  int device = 0;
  int E_l = 0;
  int64_t C = -1;
  int64_t recv_rows = 0;
  // symmetric heap: [internal: count matrix | flags][user allocations]
  char* heap = nullptr;
  size_t heap_bytes = 0;
  size_t heap_used = 0;
  size_t internal_bytes = 0;
  int64_t countmat_off = 0;
  int64_t ntokmat_off = 0;
  int64_t flags_off = 0;
  int64_t arrive_off = 0;         // fused dispatch arrival flags [E_l][EP+1] (NEXT-1)
  cudaIpcMemHandle_t handle;
  char* peer_base[MOE_MAX_EP] = {};
  bool peer_opened[MOE_MAX_EP] = {};
  bool peers_ready = false;
  // device scratch
  int32_t* d_err = nullptr;
  int32_t* d_done = nullptr;
  int32_t* d_scratch = nullptr;   // permute workspace
  int32_t* d_dedup_scratch = nullptr;   // dedup pairs workspace (masks, block bases, ticket)
  int32_t* d_rows_T = nullptr;    // one int32 = T_local (router GEMM group size)
  int32_t* d_disp_work = nullptr; // fused dispatch counters [4 + E + E_l] (zero between calls)
  int32_t* d_slot_of_row = nullptr; // [T*k] send-layout row -> slot t*k+j (moe_permute)
  uint16_t* d_dl_split = nullptr; // router backward: [T, 2*Ep] bf16 = [hi | lo] of dlogits
  uint16_t* d_wr2 = nullptr;      // [2*Ep, d] bf16 = [W_r; W_r] (dense dx_router path)
  float* d_dwr_part = nullptr;    // [S, 2*Ep, d] fp32 split-K partials of dW_r
  int32_t* d_split_rows = nullptr;// [S] token rows per split
  int n_split = 1;
  int Ep = 0;                     // E rounded up to 8
  int32_t* d_place = nullptr;     // [E] expert -> global slot (identity unless migrated)
  int32_t* d_expert_at = nullptr; // [E] global slot -> expert
  int gemm_sms = 0;               // SM budgets (0 = all): a GEMM and a transfer running
  int comm_sms = 0;               //   concurrently on two streams use disjoint SMs
  // symmetric allocations (heap offset, bytes) in allocation order, and their FNV-1a
  // fingerprint: every rank must allocate the same sizes in the same order (moe.h)
  std::vector<std::pair<size_t, size_t>> allocs;
  uint64_t fingerprint = 1469598103934665603ull;
  size_t device_bytes = 0;        // every cudaMalloc of the ctx (heap incl.)
};

namespace {

using moe::CommArgs;

moe_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return MOE_OK;
  fprintf(stderr, "[libmoe] CUDA error: %s\n", cudaGetErrorString(e));
  return MOE_ERR_CUDA;
}

#define MOE_TRY_CUDA(expr)                                 \
  do {                                                     \
    cudaError_t e_ = (expr);                               \
    if (e_ != cudaSuccess) return cuda_status(e_);         \
  } while (0)
// token-row buffers ([T_local, ...], [T_local*k, ...]) may be NULL when T_local == 0
#define TOKP(p) ((p) != nullptr || c->s.T_local == 0)
#define MOE_REQUIRE(cond)                                  \
  do {                                                     \
    if (!(cond)) return MOE_ERR_INVALID_ARG;               \
  } while (0)

bool shape_ok(const moe_shape* s) {
  if (!s) return false;
  if (s->ep_size != 1 && s->ep_size != 2 && s->ep_size != 4 && s->ep_size != 8) return false;
  if (s->E <= 0 || s->E > 256 || s->E % s->ep_size) return false;   // EP | E
  if (s->k < 1 || s->k > s->E || s->k > 32) return false;            // top_k <= E
  if (s->ep_rank < 0 || s->ep_rank >= s->ep_size) return false;
  if (s->d <= 0 || s->d % 64 || s->f <= 0 || s->f % 64) return false;
  if (s->T_local < 0 || s->E_shared < 0) return false;
  return true;
}

int64_t capacity_of(const moe_shape* s) {
  if (s->capacity_factor <= 0.f) return -1;
  // C = ceil(cf * k * T_r / E) in double (reading R4)
  double c = static_cast<double>(s->capacity_factor) * s->k * static_cast<double>(s->T_local) / s->E;
  int64_t ci = static_cast<int64_t>(c);
  if (static_cast<double>(ci) < c) ++ci;
  return ci;
}

int64_t recv_rows_of(const moe_shape* s) {
  const int64_t EP = s->ep_size, E_l = s->E / s->ep_size;
  int64_t rows = EP * s->T_local * (s->k < E_l ? s->k : E_l);
  const int64_t C = capacity_of(s);
  if (C >= 0 && EP * E_l * C < rows) rows = EP * E_l * C;
  rows += E_l * (MOE_ALIGN_ROWS - 1);
  return (rows + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
}

cudaStream_t st(moe_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// [p, p + bytes) lies inside ONE symmetric allocation (peers write up to `bytes` at p's
// offset into this rank's heap: an undersized buffer would let them overwrite a neighbour)
bool in_heap(const moe_ctx* c, const void* p, int64_t bytes) {
  const char* q = static_cast<const char*>(p);
  if (q < c->heap + c->internal_bytes || q >= c->heap + c->heap_bytes || bytes < 0) return false;
  const size_t off = static_cast<size_t>(q - c->heap);
  for (const auto& a : c->allocs)
    if (off >= a.first && off < a.first + (a.second ? a.second : 1))
      return off + static_cast<size_t>(bytes) <= a.first + a.second;
  return false;
}
int64_t row_bytes(const moe_ctx* c) { return static_cast<int64_t>(c->s.d) * 2; }
int64_t heap_off(const moe_ctx* c, const void* p) {
  return reinterpret_cast<const char*>(p) - c->heap;
}
// destination sizes of the collectives (rows of d bf16)
int64_t recv_bytes(const moe_ctx* c) { return c->recv_rows * row_bytes(c); }
int64_t send_bytes(const moe_ctx* c) { return c->s.T_local * c->s.k * row_bytes(c); }

CommArgs comm_args(moe_ctx* c) {
  CommArgs a;
  memset(&a, 0, sizeof(a));
  for (int q = 0; q < c->s.ep_size; ++q) a.peers.base[q] = c->peer_base[q];
  a.ep = c->s.ep_size;
  a.rank = c->s.ep_rank;
  a.E = c->s.E;
  a.E_l = c->E_l;
  a.d = c->s.d;
  a.T = c->s.T_local;
  a.k = c->s.k;
  a.flags = reinterpret_cast<uint64_t*>(c->heap + c->flags_off);
  a.flags_off = c->flags_off;
  a.countmat = reinterpret_cast<int32_t*>(c->heap + c->countmat_off);
  a.countmat_off = c->countmat_off;
  a.ntokmat = reinterpret_cast<int32_t*>(c->heap + c->ntokmat_off);
  a.ntokmat_off = c->ntokmat_off;
  a.done = c->d_done;
  a.err = c->d_err;
  a.epoch_ptr = reinterpret_cast<uint64_t*>(c->d_done + 4);
  a.blocks = c->comm_sms > 0 ? 2 * c->comm_sms : 0;
  a.place = c->d_place;
  a.expert_at = c->d_expert_at;
  return a;
}

// Alg. 2 of PAPER.md:672-706 (hill-climbing swap rebalancing) on the owners' slot loads,
// exact integer arithmetic; tie rules as oracle/migration.py (reading R16).
int rebalance_groups(std::vector<std::vector<int64_t>>& G, std::vector<std::vector<int>>& ids,
                     int T) {
  const int K = static_cast<int>(G.size());
  int c = 0;
  for (int t = 0; t < T; ++t) {
    std::vector<int64_t> s(K, 0);
    for (int k = 0; k < K; ++k)
      for (int64_t v : G[k]) s[k] += v;
    int kp = 0, km = 0;
    for (int k = 1; k < K; ++k) {
      if (s[k] > s[kp]) kp = k;   // first maximum
      if (s[k] < s[km]) km = k;   // first minimum
    }
    const int64_t delta = s[kp] - s[km];
    int bi = -1, bj = -1;
    int64_t best = 0;
    for (size_t i = 0; i < G[kp].size(); ++i)
      for (size_t j = 0; j < G[km].size(); ++j) {
        int64_t d2 = (s[kp] - G[kp][i] + G[km][j]) - (s[km] - G[km][j] + G[kp][i]);
        if (d2 < 0) d2 = -d2;
        if (d2 < delta && delta - d2 > best) {
          best = delta - d2;
          bi = static_cast<int>(i);
          bj = static_cast<int>(j);
        }
      }
    if (bi < 0) break;
    std::swap(G[kp][bi], G[km][bj]);
    std::swap(ids[kp][bi], ids[km][bj]);
    ++c;
  }
  return c;
}

moe_status set_device(moe_ctx* c) { return cuda_status(cudaSetDevice(c->device)); }

// CTA-pair (cta_group::2) tiles for the expert GEMMs unless MOE_GEMM_PAIR=0 (A/B testing).
int gemm_pair() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_GEMM_PAIR");
    v = (e && e[0] == '0') ? 1 : 2;
  }
  return v;
}

int pick_bn(int n) {
  if (n % 256 == 0) return 256;
  if (n % 128 == 0) return 128;
  return 64;
}

}  // namespace

extern "C" {

const char* moe_status_string(moe_status s) {
  switch (s) {
    case MOE_OK: return "MOE_OK";
    case MOE_ERR_INVALID_ARG: return "MOE_ERR_INVALID_ARG";
    case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
    case MOE_ERR_NOT_SYMMETRIC: return "MOE_ERR_NOT_SYMMETRIC";
    case MOE_ERR_OUT_OF_MEMORY: return "MOE_ERR_OUT_OF_MEMORY";
    case MOE_ERR_RECV_OVERFLOW: return "MOE_ERR_RECV_OVERFLOW";
    case MOE_ERR_TIMEOUT: return "MOE_ERR_TIMEOUT";
    case MOE_ERR_NOT_READY: return "MOE_ERR_NOT_READY";
  }
  return "MOE_ERR_UNKNOWN";
}

int64_t moe_capacity(const moe_shape* s) { return shape_ok(s) ? capacity_of(s) : -2; }
int64_t moe_recv_rows_max(const moe_shape* s) { return shape_ok(s) ? recv_rows_of(s) : -1; }
int64_t moe_layout_ints(const moe_shape* s) {
  if (!shape_ok(s)) return -1;
  const int64_t E_l = s->E / s->ep_size;
  return static_cast<int64_t>(s->ep_size) * s->E + 2 * E_l + 1;
}
int64_t moe_dedup_pair_rows_max(const moe_shape* s) {
  if (!shape_ok(s)) return -1;
  return s->T_local * (s->k < s->ep_size ? s->k : s->ep_size);
}
int64_t moe_dedup_token_rows_max(const moe_shape* s) {
  if (!shape_ok(s)) return -1;
  const int64_t a = s->ep_size * s->T_local, b = recv_rows_of(s);
  return a < b ? a : b;
}
int64_t moe_layout_offset(const moe_shape* s, int field) {
  if (!shape_ok(s)) return -1;
  const int64_t E_l = s->E / s->ep_size, base = static_cast<int64_t>(s->ep_size) * s->E;
  switch (field) {
    case MOE_LAYOUT_COUNTS_ALL: return 0;
    case MOE_LAYOUT_EXPERT_ROWS: return base;
    case MOE_LAYOUT_SEG_BASE: return base + E_l;
  }
  return -1;
}

// cudaMalloc that adds the size to the ctx's device-memory account (moe_ctx_device_bytes)
cudaError_t ctx_malloc(moe_ctx* c, void* pp, size_t bytes) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(pp), bytes);
  if (e == cudaSuccess) c->device_bytes += bytes;
  return e;
}

moe_status moe_ctx_create(moe_ctx** out, const moe_shape* shape, int device, size_t symm_heap_bytes) {
  MOE_REQUIRE(out && shape_ok(shape));
  *out = nullptr;
  moe_ctx* c = new (std::nothrow) moe_ctx();
  if (!c) return MOE_ERR_OUT_OF_MEMORY;
  c->s = *shape;
  c->device = device;
  c->E_l = shape->E / shape->ep_size;
  c->C = capacity_of(shape);
  c->recv_rows = recv_rows_of(shape);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete c; return cuda_status(e); }
  const int EP = shape->ep_size;
  c->countmat_off = 0;
  c->ntokmat_off = ((2 * EP * shape->E * 4) + 255) / 256 * 256;
  c->flags_off = c->ntokmat_off + ((2 * EP * EP * 4) + 255) / 256 * 256;
  c->arrive_off = c->flags_off + ((moe::kNumSlots * EP * 8) + 255) / 256 * 256;
  c->internal_bytes =
      ((c->arrive_off + static_cast<int64_t>(c->E_l) * (EP + 1) * 8) + 4095) / 4096 * 4096;
  c->heap_bytes = c->internal_bytes + (symm_heap_bytes + 255) / 256 * 256;
  c->heap_used = c->internal_bytes;
  e = ctx_malloc(c, &c->heap, c->heap_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->heap, 0, c->internal_bytes);
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_err, 16);
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, 16);
  // [0] last-block counter, [1] counts ticket, [4..5] = uint64 collective epoch
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_done, 32);
  if (e == cudaSuccess) e = cudaMemset(c->d_done, 0, 32);
  const int64_t scratch = moe::permute_scratch_ints(shape->T_local, shape->k, shape->E);
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_scratch, scratch * 4);
  if (e == cudaSuccess) e = cudaMemset(c->d_scratch, 0, scratch * 4);   // incl. the block ticket
  const int64_t dscratch = moe::dedup_scratch_ints(shape->T_local, shape->ep_size);
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_dedup_scratch, dscratch * 4);
  if (e == cudaSuccess) e = cudaMemset(c->d_dedup_scratch, 0, dscratch * 4);
  const size_t work_bytes = static_cast<size_t>(4 + shape->E + c->E_l) * 4;
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_disp_work, work_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->d_disp_work, 0, work_bytes);
  if (e == cudaSuccess)
    e = ctx_malloc(c, &c->d_slot_of_row,
                   static_cast<size_t>(shape->T_local > 0 ? shape->T_local * shape->k : 1) * 4);
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_rows_T, 16);
  int32_t tl = static_cast<int32_t>(shape->T_local);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_rows_T, &tl, 4, cudaMemcpyHostToDevice);
  c->Ep = (shape->E + 7) / 8 * 8;
  const int64_t Tl = shape->T_local > 0 ? shape->T_local : 1;
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_dl_split, static_cast<size_t>(Tl) * 2 * c->Ep * 2);
  if (e == cudaSuccess) e = ctx_malloc(c, &c->d_wr2, static_cast<size_t>(2) * c->Ep * shape->d * 2);
  // dW_r = x^T dl has K = T tokens and only E x d outputs: split K into S 128-row-aligned
  // token chunks (one K-grouped GEMM group each) so the GPU fills; partials summed in order.
  {
    int64_t S = Tl / 1024;
    S = S < 1 ? 1 : (S > 16 ? 16 : S);
    int64_t chunk = ((Tl + S - 1) / S + MOE_ALIGN_ROWS - 1) / MOE_ALIGN_ROWS * MOE_ALIGN_ROWS;
    S = (Tl + chunk - 1) / chunk;
    int32_t rows[16];
    for (int64_t i = 0; i < S; ++i) {
      const int64_t r = Tl - i * chunk;
      rows[i] = static_cast<int32_t>(r < chunk ? r : chunk);
    }
    if (shape->T_local == 0) rows[0] = 0;
    c->n_split = static_cast<int>(S);
    if (e == cudaSuccess) e = ctx_malloc(c, &c->d_split_rows, 16 * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_split_rows, rows, S * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = ctx_malloc(c, &c->d_dwr_part, static_cast<size_t>(S) * 2 * c->Ep * shape->d * sizeof(float));
  }
  {
    std::vector<int32_t> ident(shape->E);
    for (int i = 0; i < shape->E; ++i) ident[i] = i;
    if (e == cudaSuccess) e = ctx_malloc(c, &c->d_place, shape->E * sizeof(int32_t));
    if (e == cudaSuccess) e = ctx_malloc(c, &c->d_expert_at, shape->E * sizeof(int32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_place, ident.data(), shape->E * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_expert_at, ident.data(), shape->E * sizeof(int32_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && EP > 1) e = cudaIpcGetMemHandle(&c->handle, c->heap);
  if (e != cudaSuccess) {
    moe_ctx_destroy(c);
    return cuda_status(e);
  }
  c->peer_base[shape->ep_rank] = c->heap;
  if (EP == 1) c->peers_ready = true;
  *out = c;
  return MOE_OK;
}

moe_status moe_ctx_export_handle(moe_ctx* c, void* handle_out) {
  MOE_REQUIRE(c && handle_out);
  static_assert(sizeof(cudaIpcMemHandle_t) == MOE_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &c->handle, MOE_IPC_HANDLE_BYTES);
  return MOE_OK;
}

moe_status moe_ctx_open_peers(moe_ctx* c, const void* handles) {
  MOE_REQUIRE(c && (handles || c->s.ep_size == 1));
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  const char* h = static_cast<const char*>(handles);
  for (int q = 0; q < c->s.ep_size; ++q) {
    if (q == c->s.ep_rank || c->peer_opened[q]) continue;
    cudaIpcMemHandle_t hq;
    memcpy(&hq, h + q * MOE_IPC_HANDLE_BYTES, MOE_IPC_HANDLE_BYTES);
    void* p = nullptr;
    MOE_TRY_CUDA(cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess));
    c->peer_base[q] = static_cast<char*>(p);
    c->peer_opened[q] = true;
  }
  c->peers_ready = true;
  return MOE_OK;
}

moe_status moe_symm_alloc(moe_ctx* c, size_t bytes, void** ptr) {
  MOE_REQUIRE(c && ptr);
  const size_t sz = (bytes + 255) / 256 * 256;
  if (c->heap_used + sz > c->heap_bytes) return MOE_ERR_OUT_OF_MEMORY;
  *ptr = c->heap + c->heap_used;
  c->allocs.emplace_back(c->heap_used, bytes);
  for (uint64_t v : {static_cast<uint64_t>(c->heap_used), static_cast<uint64_t>(bytes)})
    for (int i = 0; i < 8; ++i) {
      c->fingerprint ^= (v >> (8 * i)) & 0xffu;
      c->fingerprint *= 1099511628211ull;
    }
  c->heap_used += sz;
  return MOE_OK;
}

moe_status moe_symm_free(moe_ctx* c, void* ptr) {
  MOE_REQUIRE(c && ptr && !c->allocs.empty());
  const auto& last = c->allocs.back();
  if (static_cast<char*>(ptr) != c->heap + last.first) return MOE_ERR_INVALID_ARG;   // LIFO only
  c->heap_used = last.first;
  for (uint64_t v : {~static_cast<uint64_t>(last.first), ~static_cast<uint64_t>(last.second)})
    for (int i = 0; i < 8; ++i) {
      c->fingerprint ^= (v >> (8 * i)) & 0xffu;
      c->fingerprint *= 1099511628211ull;
    }
  c->allocs.pop_back();
  return MOE_OK;
}

moe_status moe_ctx_device_bytes(moe_ctx* c, size_t* heap_bytes, size_t* heap_used,
                                size_t* total_bytes) {
  MOE_REQUIRE(c);
  if (heap_bytes) *heap_bytes = c->heap_bytes;
  if (heap_used) *heap_used = c->heap_used;
  if (total_bytes) *total_bytes = c->device_bytes;
  return MOE_OK;
}

moe_status moe_symm_fingerprint(moe_ctx* c, uint64_t* out) {
  MOE_REQUIRE(c && out);
  *out = c->fingerprint;
  return MOE_OK;
}

moe_status moe_ctx_verify_symmetric(moe_ctx* c, const uint64_t* all) {
  MOE_REQUIRE(c && all);
  for (int q = 0; q < c->s.ep_size; ++q)
    if (all[q] != c->fingerprint) return MOE_ERR_NOT_SYMMETRIC;
  return MOE_OK;
}

moe_status moe_ctx_set_placement(moe_ctx* c, const int32_t* placement) {
  MOE_REQUIRE(c && placement);
  const int E = c->s.E;
  std::vector<int32_t> inv(E, -1);
  for (int e = 0; e < E; ++e) {
    const int32_t s = placement[e];
    if (s < 0 || s >= E || inv[s] != -1) return MOE_ERR_INVALID_ARG;  // not a permutation
    inv[s] = e;
  }
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  MOE_TRY_CUDA(cudaDeviceSynchronize());  // no kernel may still read the old placement
  MOE_TRY_CUDA(cudaMemcpy(c->d_place, placement, E * sizeof(int32_t), cudaMemcpyHostToDevice));
  MOE_TRY_CUDA(cudaMemcpy(c->d_expert_at, inv.data(), E * sizeof(int32_t), cudaMemcpyHostToDevice));
  return MOE_OK;
}

moe_status moe_migrate(moe_ctx* c, const int32_t* old_place, const int32_t* new_place,
                       const void* src, void* dst, size_t bytes_per_expert, moe_stream s) {
  MOE_REQUIRE(c && old_place && new_place && src && dst);
  MOE_REQUIRE(bytes_per_expert > 0 && bytes_per_expert % 16 == 0 && c->E_l <= 256);
  const int E = c->s.E, E_l = c->E_l, r = c->s.ep_rank;
  std::vector<int> seen_o(E, 0), seen_n(E, 0);
  for (int e = 0; e < E; ++e) {
    if (old_place[e] < 0 || old_place[e] >= E || seen_o[old_place[e]]++) return MOE_ERR_INVALID_ARG;
    if (new_place[e] < 0 || new_place[e] >= E || seen_n[new_place[e]]++) return MOE_ERR_INVALID_ARG;
  }
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  const int64_t total = static_cast<int64_t>(E_l) * static_cast<int64_t>(bytes_per_expert);
  if (!in_heap(c, src, total) || !in_heap(c, dst, total)) return MOE_ERR_NOT_SYMMETRIC;
  const char* ps = static_cast<const char*>(src);
  const char* pd = static_cast<const char*>(dst);
  if (ps < pd + total && pd < ps + total) return MOE_ERR_INVALID_ARG;   // overlap
  moe::MigrateList ml;
  ml.n = 0;
  for (int e = 0; e < E; ++e) {
    if (old_place[e] / E_l != r) continue;   // this rank pushes the experts it holds now
    ml.src_slot[ml.n] = static_cast<int16_t>(old_place[e] % E_l);
    ml.dst_rank[ml.n] = static_cast<int16_t>(new_place[e] / E_l);
    ml.dst_slot[ml.n] = static_cast<int16_t>(new_place[e] % E_l);
    ++ml.n;
  }
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  CommArgs a = comm_args(c);
  return cuda_status(moe::launch_migrate(a, ml, src, heap_off(c, dst),
                                         static_cast<int64_t>(bytes_per_expert), st(s)));
}

moe_status moe_all_to_all(moe_ctx* c, const void* send, void* recv, size_t bytes_per_peer,
                          moe_stream s) {
  MOE_REQUIRE(c && send && recv && bytes_per_peer % 16 == 0);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  const int64_t total = static_cast<int64_t>(bytes_per_peer) * c->s.ep_size;
  if (!in_heap(c, recv, total)) return MOE_ERR_NOT_SYMMETRIC;
  if (bytes_per_peer == 0) return MOE_OK;
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  CommArgs a = comm_args(c);
  return cuda_status(moe::launch_all_to_all(a, send, heap_off(c, recv),
                                            static_cast<int64_t>(bytes_per_peer), st(s)));
}

moe_status moe_load_imbalance(const int64_t* loads, const int32_t* placement, int32_t E,
                              int32_t ep, double* out) {
  MOE_REQUIRE(loads && placement && out && E > 0 && ep > 0 && E % ep == 0);
  const int E_l = E / ep;
  std::vector<int64_t> s(ep, 0);
  int64_t tot = 0;
  for (int e = 0; e < E; ++e) {
    if (placement[e] < 0 || placement[e] >= E || loads[e] < 0) return MOE_ERR_INVALID_ARG;
    s[placement[e] / E_l] += loads[e];
    tot += loads[e];
  }
  int64_t mx = 0;
  for (int q = 0; q < ep; ++q) mx = s[q] > mx ? s[q] : mx;
  *out = tot == 0 ? 1.0 : static_cast<double>(mx) * ep / static_cast<double>(tot);
  return MOE_OK;
}

moe_status moe_rebalance(const int64_t* loads, int32_t E, int32_t ep, int32_t max_iters,
                         int32_t* placement, int32_t* n_swaps) {
  MOE_REQUIRE(loads && placement && E > 0 && ep > 0 && E % ep == 0 && max_iters >= 0);
  const int E_l = E / ep;
  std::vector<int32_t> expert_at(E, -1);
  for (int e = 0; e < E; ++e) {
    if (placement[e] < 0 || placement[e] >= E || expert_at[placement[e]] != -1)
      return MOE_ERR_INVALID_ARG;
    expert_at[placement[e]] = e;
  }
  std::vector<std::vector<int64_t>> G(ep, std::vector<int64_t>(E_l));
  std::vector<std::vector<int>> ids(ep, std::vector<int>(E_l));
  for (int q = 0; q < ep; ++q)
    for (int el = 0; el < E_l; ++el) {
      ids[q][el] = expert_at[q * E_l + el];
      G[q][el] = loads[ids[q][el]];
    }
  const int c = rebalance_groups(G, ids, max_iters);
  for (int q = 0; q < ep; ++q)
    for (int el = 0; el < E_l; ++el) placement[ids[q][el]] = q * E_l + el;
  if (n_swaps) *n_swaps = c;
  return MOE_OK;
}

moe_status moe_ctx_set_sm_limits(moe_ctx* c, int gemm_sms, int comm_sms) {
  MOE_REQUIRE(c && gemm_sms >= 0 && comm_sms >= 0);
  c->gemm_sms = gemm_sms;
  c->comm_sms = comm_sms;
  return MOE_OK;
}

moe_status moe_ctx_get_device_error(moe_ctx* c) {
  MOE_REQUIRE(c);
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  MOE_TRY_CUDA(cudaDeviceSynchronize());
  int32_t v = 0;
  MOE_TRY_CUDA(cudaMemcpy(&v, c->d_err, 4, cudaMemcpyDeviceToHost));
  if (v == moe::kDevTimeout) return MOE_ERR_TIMEOUT;
  if (v == moe::kDevOverflow) return MOE_ERR_RECV_OVERFLOW;
  return MOE_OK;
}

moe_status moe_ctx_destroy(moe_ctx* c) {
  if (!c) return MOE_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < MOE_MAX_EP; ++q)
    if (c->peer_opened[q]) cudaIpcCloseMemHandle(c->peer_base[q]);
  cudaFree(c->heap);
  cudaFree(c->d_err);
  cudaFree(c->d_done);
  cudaFree(c->d_scratch);
  cudaFree(c->d_dedup_scratch);
  cudaFree(c->d_rows_T);
  cudaFree(c->d_disp_work);
  cudaFree(c->d_slot_of_row);
  cudaFree(c->d_dl_split);
  cudaFree(c->d_wr2);
  cudaFree(c->d_dwr_part);
  cudaFree(c->d_split_rows);
  cudaFree(c->d_place);
  cudaFree(c->d_expert_at);
  delete c;
  return MOE_OK;
}

// ---------------------------------------------------------------- F0 / B0
moe_status moe_router_logits(moe_ctx* c, const moe_bf16* x, const moe_bf16* w_r,
                             const float* bias, float* logits, moe_stream s) {
  MOE_REQUIRE(c && TOKP(x) && w_r && TOKP(logits));
  if (c->s.T_local == 0) return MOE_OK;
  moe::GemmProblem g;
  g.epi = moe::kEpiF32Rows;
  const int E = c->s.E;
  g.BN = E <= 16 ? 16 : E <= 64 ? 64 : E <= 128 ? 128 : 256;
  g.a_ptr = x; g.a_rows = c->s.T_local; g.a_cols = c->s.d; g.a_ld = c->s.d;
  g.b_ptr = w_r; g.b_rows = E; g.b_cols = c->s.d; g.b_ld = c->s.d;
  g.b_group_stride = 0;
  g.N = E; g.K = c->s.d;
  g.group_rows = c->d_rows_T; g.n_groups = 1; g.rows_cap = c->s.T_local;
  g.out = logits; g.ld_out = E;
  g.bias = bias;
  return cuda_status(moe::launch_grouped_gemm(g, st(s)));
}

moe_status moe_router_logits_bwd(moe_ctx* c, const moe_bf16* x, const moe_bf16* w_r,
                                 const float* dlogits, float* dx_router, float* dw_r,
                                 int accumulate, moe_stream s) {
  MOE_REQUIRE(c && TOKP(x) && w_r && TOKP(dlogits) && (dx_router || dw_r));
  const int64_t T = c->s.T_local;
  const int d = c->s.d, E = c->s.E, Ep = c->Ep;
  if (T == 0) {
    if (dw_r && !accumulate) MOE_TRY_CUDA(cudaMemsetAsync(dw_r, 0, sizeof(float) * E * d, st(s)));
    return MOE_OK;
  }
  // dl = hi + lo (bf16 each) as one [T, 2*Ep] tensor: one tensor-core GEMM per output
  MOE_TRY_CUDA(moe::launch_split_hilo(dlogits, T, E, Ep, c->d_dl_split, st(s)));
  if (dx_router) {  // dx_router[T, d] = [hi | lo] . [W_r; W_r]   (K-concatenation)
    MOE_TRY_CUDA(moe::launch_stack_wr(w_r, E, Ep, d, c->d_wr2, st(s)));
    moe::GemmProblem g;
    g.epi = moe::kEpiF32Rows;
    g.BN = pick_bn(d);
    g.b_mn = true;
    g.a_ptr = c->d_dl_split; g.a_rows = T; g.a_cols = 2 * Ep; g.a_ld = 2 * Ep;
    g.b_ptr = c->d_wr2; g.b_rows = 2 * Ep; g.b_cols = d; g.b_ld = d;
    g.b_group_stride = 0;
    g.N = d; g.K = (2 * Ep + 63) / 64 * 64;
    g.group_rows = c->d_rows_T; g.n_groups = 1; g.rows_cap = T;
    g.out = dx_router; g.ld_out = d;
    MOE_TRY_CUDA(moe::launch_grouped_gemm(g, st(s)));
  }
  if (dw_r) {  // [hi | lo]^T x over S token chunks -> [S, 2*Ep, d] partials -> ordered sum
    moe::GemmProblem g;
    g.epi = moe::kEpiF32Group;
    g.BN = pick_bn(d);
    g.a_mn = true; g.b_mn = true;
    g.a_ptr = c->d_dl_split; g.a_rows = T; g.a_cols = 2 * Ep; g.a_ld = 2 * Ep;
    g.b_ptr = x; g.b_rows = T; g.b_cols = d; g.b_ld = d;
    g.M = 2 * Ep; g.N = d;
    g.group_rows = c->d_split_rows; g.n_groups = c->n_split; g.rows_cap = T;
    g.out = c->d_dwr_part;
    MOE_TRY_CUDA(moe::launch_grouped_gemm(g, st(s)));
    MOE_TRY_CUDA(moe::launch_sum_partials(c->d_dwr_part, c->n_split, E, Ep, d, dw_r, accumulate, st(s)));
  }
  return MOE_OK;
}

moe_status moe_permute_bwd_router(moe_ctx* c, const moe_bf16* dxs, const int32_t* dest_row,
                                  const int32_t* topk_idx, const float* dlogits,
                                  const moe_bf16* w_r, const moe_bf16* dx_extra, moe_bf16* dx,
                                  moe_stream s) {
  MOE_REQUIRE(c && TOKP(dxs) && TOKP(dest_row) && TOKP(topk_idx) && TOKP(dlogits) && w_r && TOKP(dx));
  MOE_REQUIRE(c->s.k > 1);  // k = 1 has a dense router gradient (full softmax)
  return cuda_status(moe::launch_permute_bwd_router(dxs, dest_row, topk_idx, dlogits, w_r, dx_extra,
                                                    c->s.T_local, c->s.d, c->s.E, c->s.k, dx, st(s)));
}

// ---------------------------------------------------------------- F1 / B1
moe_status moe_route(moe_ctx* c, const float* logits, int32_t* topk_idx, float* gates, moe_stream s) {
  MOE_REQUIRE(c && TOKP(logits) && TOKP(topk_idx) && TOKP(gates));
  return cuda_status(moe::launch_route(logits, c->s.T_local, c->s.E, c->s.k, topk_idx, gates, st(s)));
}

moe_status moe_route_bwd(moe_ctx* c, const float* logits, const int32_t* topk_idx, const float* gates,
                         const float* dgates, float* dlogits, moe_stream s) {
  MOE_REQUIRE(c && TOKP(topk_idx) && TOKP(gates) && TOKP(dgates) && TOKP(dlogits) && (TOKP(logits) || c->s.k > 1));
  return cuda_status(moe::launch_route_bwd(logits, topk_idx, gates, dgates, c->s.T_local, c->s.E,
                                           c->s.k, dlogits, st(s)));
}

// ---------------------------------------------------------------- F2 / B2
moe_status moe_permute(moe_ctx* c, const moe_bf16* x, const int32_t* topk_idx, int32_t* counts,
                       int32_t* dest_row, moe_bf16* xs, moe_stream s) {
  MOE_REQUIRE(c && TOKP(x) && TOKP(topk_idx) && counts && TOKP(dest_row));   // xs NULL: indices only
  return cuda_status(moe::launch_permute(x, topk_idx, c->s.T_local, c->s.d, c->s.E, c->s.k, c->C,
                                         counts, dest_row, xs, c->d_scratch, st(s), nullptr,
                                         nullptr, 0, c->d_slot_of_row));
}

moe_status moe_permute_dispatch_local(moe_ctx* c, const moe_bf16* x, const int32_t* topk_idx,
                                      int32_t* counts, int32_t* dest_row, int32_t* layout,
                                      moe_bf16* xr, moe_stream s) {
  MOE_REQUIRE(c && TOKP(x) && TOKP(topk_idx) && counts && TOKP(dest_row) && layout && xr);
  MOE_REQUIRE(c->s.ep_size == 1);
  if (set_device(c) != MOE_OK) return MOE_ERR_CUDA;
  const int64_t pad_max = static_cast<int64_t>(c->E_l) * (MOE_ALIGN_ROWS - 1);
  return cuda_status(moe::launch_permute(x, topk_idx, c->s.T_local, c->s.d, c->s.E, c->s.k, c->C,
                                         counts, dest_row, xr, c->d_scratch, st(s), layout,
                                         c->d_expert_at, pad_max));
}

moe_status moe_unpermute(moe_ctx* c, const moe_bf16* rows, const float* gates,
                         const int32_t* dest_row, const moe_bf16* y_extra, moe_bf16* y,
                         moe_stream s) {
  MOE_REQUIRE(c && rows && TOKP(gates) && TOKP(dest_row) && TOKP(y));
  return cuda_status(moe::launch_unpermute(rows, gates, dest_row, y_extra, c->s.T_local, c->s.d,
                                           c->s.k, y, st(s)));
}

moe_status moe_combine_bwd_local(moe_ctx* c, const moe_bf16* dy, const float* gates,
                                 const int32_t* dest_row, const moe_bf16* out,
                                 const int32_t* layout, float* dgates, moe_bf16* dout_r,
                                 moe_stream s) {
  MOE_REQUIRE(c && TOKP(dy) && TOKP(gates) && TOKP(dest_row) && out && layout && TOKP(dgates) &&
              dout_r);
  MOE_REQUIRE(c->s.ep_size == 1);
  const int64_t pad_max = static_cast<int64_t>(c->E_l) * (MOE_ALIGN_ROWS - 1);
  return cuda_status(moe::launch_combine_bwd_local(dy, gates, dest_row, out, layout, c->s.T_local,
                                                   c->s.d, c->s.k, c->s.E, pad_max, dgates,
                                                   dout_r, st(s)));
}

moe_status moe_permute_bwd(moe_ctx* c, const moe_bf16* dxs, const int32_t* dest_row,
                           const float* dx_acc, const moe_bf16* dx_extra, moe_bf16* dx, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dxs) && TOKP(dest_row) && TOKP(dx));
  return cuda_status(moe::launch_permute_bwd(dxs, dest_row, dx_acc, dx_extra, c->s.T_local, c->s.d,
                                             c->s.k, dx, st(s)));
}

// ---------------------------------------------------------------- F3 / B3
moe_status moe_dispatch_range(moe_ctx* c, const moe_bf16* xs, const int32_t* counts, int32_t* layout,
                              moe_bf16* xr, int32_t slot_begin, int32_t slot_end, moe_stream s) {
  MOE_REQUIRE(c && TOKP(xs) && layout && xr && (counts || slot_begin > 0));
  MOE_REQUIRE(slot_begin >= 0 && slot_begin < slot_end && slot_end <= c->E_l);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, xr, recv_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int64_t dst_off = reinterpret_cast<const char*>(xr) - c->heap;
  return cuda_status(moe::launch_dispatch(a, counts, layout, c->recv_rows, xs, dst_off, xr,
                                          slot_begin, slot_end, st(s)));
}

moe_status moe_dispatch(moe_ctx* c, const moe_bf16* xs, const int32_t* counts, int32_t* layout,
                        moe_bf16* xr, moe_stream s) {
  MOE_REQUIRE(c && counts);
  return moe_dispatch_range(c, xs, counts, layout, xr, 0, c->E_l, s);
}

moe_status moe_dispatch_bwd(moe_ctx* c, const moe_bf16* dxr, const int32_t* layout, moe_bf16* dxs,
                            moe_stream s) {
  MOE_REQUIRE(c && dxr && layout && TOKP(dxs));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dxs, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int64_t dst_off = reinterpret_cast<const char*>(dxs) - c->heap;
  return cuda_status(moe::launch_reverse_transfer(a, layout, dxr, dst_off, st(s)));
}

// ---------------------------------------------------------------- F4 / B4
namespace {
// Fused reverse all-to-all target of a BF16 GEMM epilogue (nullptr: plain local store).
struct Scatter {
  const CommArgs* comm;
  int64_t off;
  const int32_t* layout;
};

// GEMM1 + SwiGLU epilogue for groups [g0, n_groups): xr -> g_u_h (G, U, H)
moe_status ffn_up(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows, int32_t g0,
                  int32_t n_groups, int64_t rows_cap, int32_t f, const moe_bf16* w_gu,
                  moe_bf16* g_u_h, moe_stream s) {
  MOE_REQUIRE(n_groups >= 1 && n_groups <= 256 && g0 >= 0 && g0 < n_groups && rows_cap >= 0 &&
              f > 0 && f % 128 == 0);
  if (rows_cap == 0) return MOE_OK;
  const int d = c->s.d;
  moe::GemmProblem g1;
  g1.epi = moe::kEpiSwiGLU;
  g1.BN = 256;
  g1.a_ptr = xr; g1.a_rows = rows_cap; g1.a_cols = d; g1.a_ld = d;
  g1.b_ptr = w_gu; g1.b_rows = static_cast<int64_t>(n_groups) * 2 * f; g1.b_cols = d; g1.b_ld = d;
  g1.b_group_stride = 2 * f; g1.b_split = f;
  g1.N = 2 * f; g1.K = d;
  g1.group_rows = group_rows; g1.n_groups = n_groups; g1.group_begin = g0; g1.rows_cap = rows_cap;
  g1.pair = gemm_pair();
  g1.max_ctas = c->gemm_sms;
  g1.out = g_u_h; g1.ld_out = 3 * static_cast<int64_t>(f); g1.f = f;
  return cuda_status(moe::launch_grouped_gemm(g1, st(s)));
}

// GEMM2: H (inside g_u_h) -> out, or straight into the sources' ys (sc, combine fused)
moe_status ffn_down(moe_ctx* c, const int32_t* group_rows, int32_t n_groups, int64_t rows_cap,
                    int32_t f, const moe_bf16* w_down, moe_bf16* g_u_h, moe_bf16* out,
                    const Scatter* sc, moe_stream s) {
  MOE_REQUIRE(n_groups >= 1 && n_groups <= 256 && rows_cap >= 0 && f > 0 && f % 128 == 0);
  if (rows_cap == 0) return MOE_OK;
  const int d = c->s.d;
  moe::GemmProblem g2;
  g2.epi = moe::kEpiBF16;
  g2.BN = pick_bn(d);
  g2.a_ptr = g_u_h + 2 * static_cast<int64_t>(f); g2.a_rows = rows_cap; g2.a_cols = f;
  g2.a_ld = 3 * static_cast<int64_t>(f);
  g2.b_ptr = w_down; g2.b_rows = static_cast<int64_t>(n_groups) * d; g2.b_cols = f; g2.b_ld = f;
  g2.b_group_stride = d;
  g2.N = d; g2.K = f;
  g2.group_rows = group_rows; g2.n_groups = n_groups; g2.rows_cap = rows_cap;
  g2.pair = gemm_pair();
  g2.max_ctas = c->gemm_sms;
  g2.out = out ? static_cast<void*>(out) : static_cast<void*>(g_u_h); g2.ld_out = d;
  if (sc) {
    g2.scatter = 1; g2.scatter_off = sc->off; g2.scatter_layout = sc->layout; g2.comm = sc->comm;
  }
  return cuda_status(moe::launch_grouped_gemm(g2, st(s)));
}

moe_status ffn_fwd(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows, int32_t n_groups,
                   int64_t rows_cap, int32_t f, const moe_bf16* w_gu, const moe_bf16* w_down,
                   moe_bf16* g_u_h, moe_bf16* out, const Scatter* sc, moe_stream s) {
  moe_status r = ffn_up(c, xr, group_rows, 0, n_groups, rows_cap, f, w_gu, g_u_h, s);
  if (r != MOE_OK) return r;
  return ffn_down(c, group_rows, n_groups, rows_cap, f, w_down, g_u_h, out, sc, s);
}
}  // namespace

moe_status moe_expert_ffn(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows, int32_t n_groups,
                          int64_t rows_cap, int32_t f, const moe_bf16* w_gu, const moe_bf16* w_down,
                          moe_bf16* g_u_h, moe_bf16* out, moe_stream s) {
  // row buffers may be NULL when rows_cap == 0 (e.g. the shared experts of a T_local = 0 rank)
  const bool r0 = rows_cap == 0;
  MOE_REQUIRE(c && (xr || r0) && group_rows && w_gu && w_down && (g_u_h || r0) && (out || r0));
  return ffn_fwd(c, xr, group_rows, n_groups, rows_cap, f, w_gu, w_down, g_u_h, out, nullptr, s);
}

namespace {
// dgrad-1: dH = dout . W_down^T (+ dSwiGLU epilogue) -> dgu, for groups [g0, n_groups)
moe_status ffn_bwd_dh(moe_ctx* c, const int32_t* group_rows, int32_t g0, int32_t n_groups,
                      int64_t rows_cap, int32_t f, const moe_bf16* w_down, const moe_bf16* g_u_h,
                      const moe_bf16* dout, moe_bf16* dgu, moe_stream s) {
  MOE_REQUIRE(n_groups >= 1 && n_groups <= 256 && g0 >= 0 && g0 < n_groups && rows_cap >= 0 &&
              f > 0 && f % 128 == 0);
  if (rows_cap == 0) return MOE_OK;
  const int d = c->s.d;
  const int64_t F = f;
  moe::GemmProblem a;
  a.epi = moe::kEpiDSwiGLU;
  // 256-column tiles also when f is an odd multiple of 128: the last n-tile is half out of
  // bounds (zero B columns, no stores) -- cheaper than every tile at 128 columns (DS-MoE
  // f = 1408: the BN = 128 dgrad-1 ran its tensor pipe 38 % of the time)
  a.BN = f >= 256 ? 256 : 128;
  a.b_mn = true;
  a.a_ptr = dout; a.a_rows = rows_cap; a.a_cols = d; a.a_ld = d;
  a.b_ptr = w_down; a.b_rows = static_cast<int64_t>(n_groups) * d; a.b_cols = f; a.b_ld = f;
  a.b_group_stride = d;
  a.N = f; a.K = d;
  a.group_rows = group_rows; a.n_groups = n_groups; a.group_begin = g0; a.rows_cap = rows_cap;
  a.pair = gemm_pair();
  a.max_ctas = c->gemm_sms;
  a.out = dgu; a.ld_out = 2 * F; a.aux = g_u_h; a.ld_aux = 3 * F; a.f = f;
  return cuda_status(moe::launch_grouped_gemm(a, st(s)));
}

// dgrad-2 (-> dxr, or straight into the sources' dxs: dispatch_bwd fused) and both wgrads
moe_status ffn_bwd_dx(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows, int32_t n_groups,
                      int64_t rows_cap, int32_t f, const moe_bf16* w_gu, const moe_bf16* g_u_h,
                      const moe_bf16* dout, const moe_bf16* dgu, moe_bf16* dxr, float* dw_gu,
                      float* dw_down, int accumulate, const Scatter* sc, moe_stream s) {
  MOE_REQUIRE(n_groups >= 1 && n_groups <= 256 && rows_cap >= 0 && f > 0 && f % 128 == 0);
  const int d = c->s.d;
  const int64_t F = f;
  if (rows_cap == 0) {
    if (!accumulate) {
      MOE_TRY_CUDA(cudaMemsetAsync(dw_gu, 0, sizeof(float) * n_groups * 2 * F * d, st(s)));
      MOE_TRY_CUDA(cudaMemsetAsync(dw_down, 0, sizeof(float) * n_groups * F * d, st(s)));
    }
    return MOE_OK;
  }
  // dgrad-2: dX = [dG dU] . W_gu  -> dxr
  moe::GemmProblem b;
  b.epi = moe::kEpiBF16;
  b.BN = pick_bn(d);
  b.b_mn = true;
  b.a_ptr = dgu; b.a_rows = rows_cap; b.a_cols = 2 * F; b.a_ld = 2 * F;
  b.b_ptr = w_gu; b.b_rows = static_cast<int64_t>(n_groups) * 2 * F; b.b_cols = d; b.b_ld = d;
  b.b_group_stride = 2 * F;
  b.N = d; b.K = 2 * f;
  b.group_rows = group_rows; b.n_groups = n_groups; b.rows_cap = rows_cap;
  b.pair = gemm_pair();
  b.max_ctas = c->gemm_sms;
  b.out = dxr ? static_cast<void*>(dxr) : const_cast<moe_bf16*>(dgu); b.ld_out = d;
  if (sc) {  // dX rows go straight back to their source ranks (dispatch_bwd fused)
    b.scatter = 1; b.scatter_off = sc->off; b.scatter_layout = sc->layout; b.comm = sc->comm;
  }
  MOE_TRY_CUDA(moe::launch_grouped_gemm(b, st(s)));
  // wgrad: dW_down[g] = dout_g^T H_g   [d, f]
  moe::GemmProblem w1;
  w1.epi = moe::kEpiF32Group;
  w1.BN = f >= 256 ? 256 : 128;   // as dgrad-1; the fp32 tensor map clips columns >= f
  w1.a_mn = true; w1.b_mn = true;
  w1.a_ptr = dout; w1.a_rows = rows_cap; w1.a_cols = d; w1.a_ld = d;
  w1.b_ptr = g_u_h + 2 * F; w1.b_rows = rows_cap; w1.b_cols = f; w1.b_ld = 3 * F;
  w1.M = d; w1.N = f;
  w1.group_rows = group_rows; w1.n_groups = n_groups; w1.rows_cap = rows_cap;
  w1.pair = gemm_pair();
  w1.max_ctas = c->gemm_sms;
  w1.out = dw_down; w1.accumulate = accumulate;
  w1.n_fastest = w1.M > w1.N;   // keep the smaller operand slab re-read from L2
  MOE_TRY_CUDA(moe::launch_grouped_gemm(w1, st(s)));
  // wgrad: dW_gu[g] = dgu_g^T X_g   [2f, d]
  moe::GemmProblem w2;
  w2.epi = moe::kEpiF32Group;
  w2.BN = pick_bn(d);
  w2.a_mn = true; w2.b_mn = true;
  w2.a_ptr = dgu; w2.a_rows = rows_cap; w2.a_cols = 2 * F; w2.a_ld = 2 * F;
  w2.b_ptr = xr; w2.b_rows = rows_cap; w2.b_cols = d; w2.b_ld = d;
  w2.M = 2 * f; w2.N = d;
  w2.group_rows = group_rows; w2.n_groups = n_groups; w2.rows_cap = rows_cap;
  w2.pair = gemm_pair();
  w2.max_ctas = c->gemm_sms;
  w2.out = dw_gu; w2.accumulate = accumulate;
  w2.n_fastest = w2.M > w2.N;
  return cuda_status(moe::launch_grouped_gemm(w2, st(s)));
}

moe_status ffn_bwd(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows, int32_t n_groups,
                   int64_t rows_cap, int32_t f, const moe_bf16* w_gu, const moe_bf16* w_down,
                   const moe_bf16* g_u_h, const moe_bf16* dout, moe_bf16* dgu, moe_bf16* dxr,
                   float* dw_gu, float* dw_down, int accumulate, const Scatter* sc, moe_stream s) {
  moe_status r = ffn_bwd_dh(c, group_rows, 0, n_groups, rows_cap, f, w_down, g_u_h, dout, dgu, s);
  if (r != MOE_OK) return r;
  return ffn_bwd_dx(c, xr, group_rows, n_groups, rows_cap, f, w_gu, g_u_h, dout, dgu, dxr, dw_gu,
                    dw_down, accumulate, sc, s);
}
}  // namespace

moe_status moe_expert_ffn_bwd(moe_ctx* c, const moe_bf16* xr, const int32_t* group_rows,
                              int32_t n_groups, int64_t rows_cap, int32_t f, const moe_bf16* w_gu,
                              const moe_bf16* w_down, const moe_bf16* g_u_h, const moe_bf16* dout,
                              moe_bf16* dgu, moe_bf16* dxr, float* dw_gu, float* dw_down,
                              int accumulate, moe_stream s) {
  const bool r0 = rows_cap == 0;
  MOE_REQUIRE(c && (xr || r0) && group_rows && w_gu && w_down && (g_u_h || r0) && (dout || r0) &&
              (dgu || r0) && (dxr || r0) && dw_gu && dw_down);
  return ffn_bwd(c, xr, group_rows, n_groups, rows_cap, f, w_gu, w_down, g_u_h, dout, dgu, dxr,
                 dw_gu, dw_down, accumulate, nullptr, s);
}

// ---------------------------------------------------------------- F4+F5+F6 / B4+B3 fused
moe_status moe_expert_ffn_up(moe_ctx* c, const moe_bf16* xr, const int32_t* layout,
                             int32_t slot_begin, int32_t slot_end, const moe_bf16* w_gu,
                             moe_bf16* g_u_h, moe_stream s) {
  MOE_REQUIRE(c && xr && layout && w_gu && g_u_h);
  MOE_REQUIRE(slot_begin >= 0 && slot_begin < slot_end && slot_end <= c->E_l);
  const int32_t* expert_rows = layout + static_cast<int64_t>(c->s.ep_size) * c->s.E;
  return ffn_up(c, xr, expert_rows, slot_begin, slot_end, c->recv_rows, c->s.f, w_gu, g_u_h, s);
}

moe_status moe_dispatch_expert_ffn_up(moe_ctx* c, const moe_bf16* xs, const int32_t* counts,
                                      int32_t* layout, moe_bf16* xr, const moe_bf16* w_gu,
                                      moe_bf16* g_u_h, moe_stream s) {
  MOE_REQUIRE(c && TOKP(xs) && counts && layout && xr && w_gu && g_u_h);
  MOE_REQUIRE(c->s.f % 128 == 0);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, xr, recv_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int d = c->s.d, f = c->s.f;
  moe::GemmProblem g1;
  g1.epi = moe::kEpiSwiGLUDisp;
  g1.BN = 256;
  g1.a_ptr = xr; g1.a_rows = c->recv_rows; g1.a_cols = d; g1.a_ld = d;
  g1.b_ptr = w_gu; g1.b_rows = static_cast<int64_t>(c->E_l) * 2 * f; g1.b_cols = d; g1.b_ld = d;
  g1.b_group_stride = 2 * f; g1.b_split = f;
  g1.N = 2 * f; g1.K = d;
  g1.n_groups = c->E_l; g1.rows_cap = c->recv_rows;
  g1.pair = gemm_pair();
  // a launch that carries a collective spins on peers: it obeys the transfer SM budget too
  // (the PP x EP executor keeps SMs free for the NCCL stage hand-offs, moe_ctx_set_sm_limits)
  g1.max_ctas = c->gemm_sms > 0 ? c->gemm_sms : c->comm_sms;
  g1.out = g_u_h; g1.ld_out = 3 * static_cast<int64_t>(f); g1.f = f;
  g1.comm = &a;
  g1.disp_src = xs; g1.disp_counts = counts; g1.disp_layout = layout;
  g1.disp_dst_off = heap_off(c, xr);
  g1.arrive_off = c->arrive_off;
  g1.disp_work = c->d_disp_work;
  return cuda_status(moe::launch_grouped_gemm(g1, st(s)));
}

moe_status moe_combine_bwd_expert_ffn_dh(moe_ctx* c, const moe_bf16* dy, const float* gates,
                                         const int32_t* dest_row, const moe_bf16* ys,
                                         const int32_t* layout, float* dgates, moe_bf16* dout_r,
                                         const moe_bf16* w_down, const moe_bf16* g_u_h,
                                         moe_bf16* dgu, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dy) && TOKP(gates) && TOKP(dest_row) && TOKP(ys) && layout && TOKP(dgates) &&
              dout_r && w_down && g_u_h && dgu);
  MOE_REQUIRE(c->s.f % 128 == 0);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dout_r, recv_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int d = c->s.d, f = c->s.f;
  const int64_t F = f;
  moe::GemmProblem g;
  g.epi = moe::kEpiDSwiGLUComb;
  g.BN = f >= 256 ? 256 : 128;   // as ffn_bwd_dh
  g.b_mn = true;
  g.a_ptr = dout_r; g.a_rows = c->recv_rows; g.a_cols = d; g.a_ld = d;
  g.b_ptr = w_down; g.b_rows = static_cast<int64_t>(c->E_l) * d; g.b_cols = f; g.b_ld = f;
  g.b_group_stride = d;
  g.N = f; g.K = d;
  g.n_groups = c->E_l; g.rows_cap = c->recv_rows;
  g.pair = gemm_pair();
  // a launch that carries a collective spins on peers: it obeys the transfer SM budget too
  // (the PP x EP executor keeps SMs free for the NCCL stage hand-offs, moe_ctx_set_sm_limits)
  g.max_ctas = c->gemm_sms > 0 ? c->gemm_sms : c->comm_sms;
  g.out = dgu; g.ld_out = 2 * F; g.aux = g_u_h; g.ld_aux = 3 * F; g.f = f;
  g.comm = &a;
  g.disp_dst_off = heap_off(c, dout_r);
  g.arrive_off = c->arrive_off;
  g.disp_work = c->d_disp_work;
  g.cb_dy = dy; g.cb_gates = gates; g.cb_ys = ys; g.cb_dgates = dgates;
  g.cb_slot_of_row = c->d_slot_of_row; g.cb_dest_row = dest_row; g.cb_layout = layout;
  return cuda_status(moe::launch_grouped_gemm(g, st(s)));
}

moe_status moe_expert_ffn_down_combine(moe_ctx* c, const int32_t* layout, const moe_bf16* w_down,
                                       moe_bf16* g_u_h, moe_bf16* ys, const float* gates,
                                       const int32_t* dest_row, const moe_bf16* y_extra,
                                       moe_bf16* y, moe_stream s) {
  MOE_REQUIRE(c && layout && w_down && g_u_h && TOKP(ys) && TOKP(gates) && TOKP(dest_row) && TOKP(y));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, ys, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const Scatter sc{&a, reinterpret_cast<const char*>(ys) - c->heap, layout};
  const int32_t* expert_rows = layout + static_cast<int64_t>(c->s.ep_size) * c->s.E;
  moe_status r = ffn_down(c, expert_rows, c->E_l, c->recv_rows, c->s.f, w_down, g_u_h, nullptr,
                          &sc, s);
  if (r != MOE_OK) return r;
  MOE_TRY_CUDA(moe::launch_wait_flags(a, moe::kSlotData, st(s)));
  return cuda_status(moe::launch_unpermute(ys, gates, dest_row, y_extra, c->s.T_local, c->s.d,
                                           c->s.k, y, st(s)));
}

moe_status moe_expert_ffn_combine(moe_ctx* c, const moe_bf16* xr, const int32_t* layout,
                                  const moe_bf16* w_gu, const moe_bf16* w_down, moe_bf16* g_u_h,
                                  moe_bf16* ys, const float* gates, const int32_t* dest_row,
                                  const moe_bf16* y_extra, moe_bf16* y, moe_stream s) {
  MOE_REQUIRE(c && xr && layout && w_gu && w_down && g_u_h && TOKP(ys) && TOKP(gates) && TOKP(dest_row) && TOKP(y));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, ys, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  moe_status r = moe_expert_ffn_up(c, xr, layout, 0, c->E_l, w_gu, g_u_h, s);
  if (r != MOE_OK) return r;
  return moe_expert_ffn_down_combine(c, layout, w_down, g_u_h, ys, gates, dest_row, y_extra, y, s);
}

moe_status moe_expert_ffn_bwd_dh(moe_ctx* c, const int32_t* layout, int32_t slot_begin,
                                 int32_t slot_end, const moe_bf16* w_down, const moe_bf16* g_u_h,
                                 const moe_bf16* dout, moe_bf16* dgu, moe_stream s) {
  MOE_REQUIRE(c && layout && w_down && g_u_h && dout && dgu);
  MOE_REQUIRE(slot_begin >= 0 && slot_begin < slot_end && slot_end <= c->E_l);
  const int32_t* expert_rows = layout + static_cast<int64_t>(c->s.ep_size) * c->s.E;
  return ffn_bwd_dh(c, expert_rows, slot_begin, slot_end, c->recv_rows, c->s.f, w_down, g_u_h,
                    dout, dgu, s);
}

moe_status moe_expert_ffn_bwd_dx_dispatch(moe_ctx* c, const moe_bf16* xr, const int32_t* layout,
                                          const moe_bf16* w_gu, const moe_bf16* g_u_h,
                                          const moe_bf16* dout, const moe_bf16* dgu, moe_bf16* dxs,
                                          float* dw_gu, float* dw_down, int accumulate,
                                          moe_stream s) {
  MOE_REQUIRE(c && xr && layout && w_gu && g_u_h && dout && dgu && TOKP(dxs) && dw_gu && dw_down);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dxs, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const Scatter sc{&a, reinterpret_cast<const char*>(dxs) - c->heap, layout};
  const int32_t* expert_rows = layout + static_cast<int64_t>(c->s.ep_size) * c->s.E;
  moe_status r = ffn_bwd_dx(c, xr, expert_rows, c->E_l, c->recv_rows, c->s.f, w_gu, g_u_h, dout,
                            dgu, nullptr, dw_gu, dw_down, accumulate, &sc, s);
  if (r != MOE_OK) return r;
  // the dX rows streamed to the sources during dgrad-2 and the two wgrad GEMMs
  return cuda_status(moe::launch_wait_flags(a, moe::kSlotData, st(s)));
}

moe_status moe_expert_ffn_bwd_dispatch(moe_ctx* c, const moe_bf16* xr, const int32_t* layout,
                                       const moe_bf16* w_gu, const moe_bf16* w_down,
                                       const moe_bf16* g_u_h, const moe_bf16* dout, moe_bf16* dgu,
                                       moe_bf16* dxs, float* dw_gu, float* dw_down, int accumulate,
                                       moe_stream s) {
  MOE_REQUIRE(c && xr && layout && w_gu && w_down && g_u_h && dout && dgu && TOKP(dxs) && dw_gu && dw_down);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dxs, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  moe_status r = moe_expert_ffn_bwd_dh(c, layout, 0, c->E_l, w_down, g_u_h, dout, dgu, s);
  if (r != MOE_OK) return r;
  return moe_expert_ffn_bwd_dx_dispatch(c, xr, layout, w_gu, g_u_h, dout, dgu, dxs, dw_gu, dw_down,
                                        accumulate, s);
}

// ---------------------------------------------------------------- F5+F6 / B6+B5
moe_status moe_combine(moe_ctx* c, const moe_bf16* out, const int32_t* layout, moe_bf16* ys,
                       const float* gates, const int32_t* dest_row, const moe_bf16* y_extra,
                       moe_bf16* y, moe_stream s) {
  MOE_REQUIRE(c && out && layout && TOKP(ys) && TOKP(gates) && TOKP(dest_row) && TOKP(y));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, ys, send_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int64_t dst_off = reinterpret_cast<const char*>(ys) - c->heap;
  MOE_TRY_CUDA(moe::launch_reverse_transfer(a, layout, out, dst_off, st(s)));
  return cuda_status(moe::launch_unpermute(ys, gates, dest_row, y_extra, c->s.T_local, c->s.d,
                                           c->s.k, y, st(s)));
}

moe_status moe_combine_bwd_range(moe_ctx* c, const moe_bf16* dy, const float* gates,
                                 const int32_t* dest_row, const moe_bf16* ys, const int32_t* layout,
                                 float* dgates, moe_bf16* dout_r, int32_t slot_begin,
                                 int32_t slot_end, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dy) && TOKP(gates) && TOKP(dest_row) && TOKP(ys) && layout && TOKP(dgates) && dout_r);
  MOE_REQUIRE(slot_begin >= 0 && slot_begin < slot_end && slot_end <= c->E_l);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dout_r, recv_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  const int64_t dst_off = reinterpret_cast<const char*>(dout_r) - c->heap;
  return cuda_status(moe::launch_combine_bwd_transfer(a, const_cast<int32_t*>(layout), dst_off,
                                                      dout_r, dest_row, gates, dy, ys, dgates,
                                                      slot_begin, slot_end, st(s)));
}

moe_status moe_combine_bwd(moe_ctx* c, const moe_bf16* dy, const float* gates, const int32_t* dest_row,
                           const moe_bf16* ys, const int32_t* layout, float* dgates, moe_bf16* dout_r,
                           moe_stream s) {
  MOE_REQUIRE(c);
  return moe_combine_bwd_range(c, dy, gates, dest_row, ys, layout, dgates, dout_r, 0, c->E_l, s);
}

}  // extern "C"

// ---------------------------------------------------------------- NEXT-4 dedup all-to-all
// Reading R18 (oracle/dedup.py): one row per (token, owner) pair crosses NVLink.
namespace {
int64_t tok_rows(const moe_ctx* c) { return moe_dedup_token_rows_max(&c->s); }
int64_t pair_rows(const moe_ctx* c) { return moe_dedup_pair_rows_max(&c->s); }
}  // namespace

moe_status moe_dedup_pairs(moe_ctx* c, const int32_t* topk_idx, const int32_t* dest_row,
                           int32_t* pdest, int32_t* ntok, moe_stream s) {
  MOE_REQUIRE(c && TOKP(topk_idx) && TOKP(dest_row) && TOKP(pdest) && ntok);
  return cuda_status(moe::launch_dedup_pairs(topk_idx, dest_row, c->d_place, c->s.T_local, c->s.k,
                                             c->E_l, c->s.ep_size, pdest, ntok,
                                             c->d_dedup_scratch, st(s)));
}

moe_status moe_dedup_dispatch(moe_ctx* c, const moe_bf16* x, const int32_t* counts,
                              const int32_t* ntok, const int32_t* pdest, const int32_t* dest_row,
                              const int32_t* topk_idx, const float* gates, int32_t* layout,
                              int32_t* dlayout, moe_bf16* xt, int32_t* rlist, float* glist,
                              moe_bf16* xr, moe_stream s) {
  MOE_REQUIRE(c && TOKP(x) && counts && ntok && TOKP(pdest) && TOKP(dest_row) && TOKP(topk_idx) && TOKP(gates) && layout &&
              dlayout && TOKP(xt) && TOKP(rlist) && TOKP(glist) && xr);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, xt, tok_rows(c) * row_bytes(c)) || !in_heap(c, rlist, tok_rows(c) * c->s.k * 4) ||
      !in_heap(c, glist, tok_rows(c) * c->s.k * 4))
    return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  MOE_TRY_CUDA(moe::launch_dedup_forward(a, 0, layout, dlayout, counts, ntok, c->recv_rows, x,
                                         pdest, dest_row, topk_idx, gates, heap_off(c, xt),
                                         heap_off(c, rlist), heap_off(c, glist), nullptr, nullptr,
                                         st(s)));
  return cuda_status(moe::launch_dedup_expand(a, 0, layout, dlayout, xt, rlist, glist, nullptr, xr,
                                              nullptr, st(s)));
}

moe_status moe_dedup_combine(moe_ctx* c, const moe_bf16* out, const int32_t* dlayout,
                             const int32_t* rlist, const float* glist, const int32_t* pdest,
                             const moe_bf16* y_extra, moe_bf16* part, moe_bf16* y, moe_stream s) {
  MOE_REQUIRE(c && out && dlayout && TOKP(rlist) && TOKP(glist) && TOKP(pdest) && TOKP(part) && TOKP(y));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, part, pair_rows(c) * row_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  MOE_TRY_CUDA(moe::launch_dedup_reduce(a, 0, dlayout, rlist, glist, out, nullptr,
                                        heap_off(c, part), 0, st(s)));
  // y[t] = bf16( sum_q part[pdest[t,q]] (q ascending) + y_extra[t] )
  return cuda_status(moe::launch_permute_bwd(part, pdest, nullptr, y_extra, c->s.T_local, c->s.d,
                                             c->s.ep_size, y, st(s)));
}

moe_status moe_dedup_combine_bwd(moe_ctx* c, const moe_bf16* dy, const int32_t* pdest,
                                 const int32_t* layout, const int32_t* dlayout,
                                 const int32_t* rlist, const float* glist, const moe_bf16* out,
                                 moe_bf16* dyt, float* dg_own, moe_bf16* dout_r, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dy) && TOKP(pdest) && layout && dlayout && TOKP(rlist) && TOKP(glist) && out && TOKP(dyt) && TOKP(dg_own) &&
              dout_r);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dyt, tok_rows(c) * row_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  MOE_TRY_CUDA(moe::launch_dedup_forward(a, 1, const_cast<int32_t*>(layout),
                                         const_cast<int32_t*>(dlayout), nullptr, nullptr, 0, dy,
                                         pdest, nullptr, nullptr, nullptr, heap_off(c, dyt), 0, 0,
                                         nullptr, nullptr, st(s)));
  return cuda_status(moe::launch_dedup_expand(a, 1, layout, dlayout, dyt, rlist, glist, out,
                                              dout_r, dg_own, st(s)));
}

moe_status moe_dedup_combine_bwd_ys(moe_ctx* c, const moe_bf16* dy, const float* gates,
                                    const int32_t* dest_row, const moe_bf16* ys,
                                    const int32_t* pdest, const int32_t* layout,
                                    const int32_t* dlayout, const int32_t* rlist,
                                    const float* glist, moe_bf16* dyt, float* dgates,
                                    moe_bf16* dout_r, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dy) && TOKP(gates) && TOKP(dest_row) && TOKP(ys) && TOKP(pdest) && layout && dlayout && TOKP(rlist) && TOKP(glist) &&
              TOKP(dyt) && TOKP(dgates) && dout_r);
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dyt, tok_rows(c) * row_bytes(c))) return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  MOE_TRY_CUDA(moe::launch_dedup_forward(a, 1, const_cast<int32_t*>(layout),
                                         const_cast<int32_t*>(dlayout), nullptr, nullptr, 0, dy,
                                         pdest, dest_row, nullptr, gates, heap_off(c, dyt), 0, 0,
                                         ys, dgates, st(s)));
  return cuda_status(moe::launch_dedup_expand(a, 1, layout, dlayout, dyt, rlist, glist, nullptr,
                                              dout_r, nullptr, st(s)));
}

moe_status moe_dedup_dispatch_bwd(moe_ctx* c, const moe_bf16* dxr, const int32_t* dlayout,
                                  const int32_t* rlist, const float* dg_own, const int32_t* pdest,
                                  const int32_t* dest_row, const int32_t* topk_idx,
                                  moe_bf16* dxpart, float* dgpart, float* dgates, moe_stream s) {
  MOE_REQUIRE(c && dxr && dlayout && TOKP(rlist) && TOKP(dg_own) && TOKP(pdest) && TOKP(dest_row) && TOKP(topk_idx) && TOKP(dxpart) &&
              TOKP(dgpart) && TOKP(dgates));
  if (!c->peers_ready) return MOE_ERR_NOT_READY;
  if (!in_heap(c, dxpart, pair_rows(c) * row_bytes(c)) ||
      !in_heap(c, dgpart, pair_rows(c) * c->s.k * 4))
    return MOE_ERR_NOT_SYMMETRIC;
  CommArgs a = comm_args(c);
  MOE_TRY_CUDA(moe::launch_dedup_reduce(a, 1, dlayout, rlist, nullptr, dxr, dg_own,
                                        heap_off(c, dxpart), heap_off(c, dgpart), st(s)));
  return cuda_status(moe::launch_dedup_dgates(dest_row, topk_idx, pdest, c->d_place, c->E_l,
                                              c->s.ep_size, dgpart, c->s.T_local, c->s.k, dgates,
                                              st(s)));
}

moe_status moe_dedup_permute_bwd_router(moe_ctx* c, const moe_bf16* dxpart, const int32_t* pdest,
                                        const int32_t* topk_idx, const float* dlogits,
                                        const moe_bf16* w_r, const moe_bf16* dx_extra,
                                        moe_bf16* dx, moe_stream s) {
  MOE_REQUIRE(c && TOKP(dxpart) && TOKP(pdest) && TOKP(topk_idx) && TOKP(dlogits) && w_r && TOKP(dx));
  MOE_REQUIRE(c->s.k > 1);
  return cuda_status(moe::launch_permute_bwd_router_rows(dxpart, pdest, c->s.ep_size, topk_idx,
                                                         dlogits, w_r, dx_extra, c->s.T_local,
                                                         c->s.d, c->s.E, c->s.k, dx, st(s)));
}

// ---------------------------------------------------------------- NEXT-3 PP x EP executor
// 1F1B op order of one pipeline stage (reading R19): w = min(PP-i-1, M)
// warm-up forwards, then one forward + one backward while forwards remain, then the
// remaining backwards; micro-batches ascending.  Host code: the executor asks for it once.
moe_status moe_pipeline_1f1b(int32_t pp, int32_t stage, int32_t n_micro, int32_t* ops,
                             int32_t max_ops, int32_t* n_ops) {
  MOE_REQUIRE(pp >= 1 && stage >= 0 && stage < pp && n_micro >= 1 && ops && n_ops);
  MOE_REQUIRE(max_ops >= 2 * n_micro);
  const int32_t w = (pp - stage - 1) < n_micro ? (pp - stage - 1) : n_micro;
  int32_t n = 0, nf = 0, nb = 0;
  auto put = [&](int32_t kind, int32_t m) {
    ops[2 * n] = kind;
    ops[2 * n + 1] = m;
    ++n;
  };
  for (; nf < w; ++nf) put(MOE_PIPE_FORWARD, nf);
  while (nf < n_micro) {
    put(MOE_PIPE_FORWARD, nf++);
    put(MOE_PIPE_BACKWARD, nb++);
  }
  while (nb < n_micro) put(MOE_PIPE_BACKWARD, nb++);
  *n_ops = n;
  return MOE_OK;
}
