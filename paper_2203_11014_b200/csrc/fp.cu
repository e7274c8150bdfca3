// fp.cu — NEXT#4: the feature processing layer in front of the DHEN stack ("we use the same feature
// processing layer in DLRM"; readings R32-R34 in DESIGN.md §3).
//
//   sparse: X0[b][n_dtok + t] = sum_{e in bag(b, t)} E_t[ids[e]]          (one pooled token per table)
//   dense:  H_0 = dense, H_k = relu(H_{k-1} W_k^T + b_k), X0[b][0 .. n_dtok) = H_L[b] as n_dtok d-vectors
//   backward + SGD: E_t[r] -= lr sum_{occurrences of r} dX0[b][n_dtok + t]; the bottom MLP by GEMMs + SGD.
//
// B200 layout: every table lives in one fp32 buffer [sum_t R_t][d] (row r of table t at row_base[t] + r);
// the forward is a gather (one warp per bag, 16-B lanes across the row, four rows in flight per warp), the
// backward sorts the (row, bag) occurrence pairs once (CUB radix sort: stable, so equal rows keep their
// sample order), compacts the run heads (CUB select), and a persistent kernel gives each run of equal rows
// to one warp, which sums its dX0 tokens in that order (eight rows in flight) and applies the SGD update in
// place -- deterministic, no atomics, no dense gradient table.  The bottom MLP runs on the library's
// tcgen05 GEMM engine with bias + ReLU epilogues (last layer written straight into X0's dense tokens) and
// ReLU-mask epilogues in the backward.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/dhen.h"
#include "gemm.h"
#include "kernels.h"

namespace dhen {
dhen_status fail_msg(dhen_status s, const char* msg);   // runtime.cu: sets dhen_last_error()
}
using namespace dhen;

namespace {

dhen_status ffail(dhen_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return fail_msg(s, buf);
}
#define FCK(call)                                                                                          \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess) return ffail(DHEN_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

template <typename T> __device__ __forceinline__ void st4(T* p, float4 v);
template <> __device__ __forceinline__ void st4<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
template <> __device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}
template <typename T> __device__ __forceinline__ float4 ld4(const T* p);
template <> __device__ __forceinline__ float4 ld4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <> __device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xffff0000u));
}

// Forward gather: warp = bag (b, t); lane owns columns 4 lane + 128 c (c < d / 128, d <= 512); four rows in
// flight, summed in list order.  Ids outside [0, R_t) are skipped and counted in *bad.
template <typename OT>
__global__ void __launch_bounds__(256) emb_fwd_k(const float* __restrict__ tab, const long long* __restrict__ rbase,
                                                 const long long* __restrict__ rows, const int* __restrict__ ids,
                                                 const int* __restrict__ off, int B, int ns, int nd, int d, int m0,
                                                 OT* __restrict__ x0, int* bad) {
  pdl_entry();
  const int bag = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (bag >= B * ns) return;
  const int b = bag / ns, t = bag - b * ns;
  const int lo = off[bag], hi = off[bag + 1];
  const float* T = tab + rbase[t] * (long long)d;
  const long long R = rows[t];
  const int nc = (d + 127) >> 7;
  float4 acc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int e = lo; e < hi; e += 4) {
    long long r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = e + u < hi ? (long long)__ldg(ids + e + u) : -1;
      if (e + u < hi && (r[u] < 0 || r[u] >= R)) {
        if (lane == 0) atomicAdd(bad, 1);
        r[u] = -1;
      }
    }
    float4 v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = 128 * c + 4 * lane;
        v[u][c] = (r[u] >= 0 && c < nc && col < d) ? __ldg(reinterpret_cast<const float4*>(T + r[u] * d + col))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c].x += v[u][c].x; acc[c].y += v[u][c].y; acc[c].z += v[u][c].z; acc[c].w += v[u][c].w;
      }
  }
  OT* dst = x0 + ((long long)b * m0 + nd + t) * d;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int col = 128 * c + 4 * lane;
    if (c < nc && col < d) st4<OT>(dst + col, acc[c]);
  }
}

// Backward, step 1: the occurrence keys (global table row; invalid ids -> the sentinel total_rows, sorted last)
// and their bag ids, in list order.
__global__ void __launch_bounds__(256) emb_keys_k(const long long* __restrict__ rbase, const long long* __restrict__ rows,
                                                  const int* __restrict__ ids, const int* __restrict__ off, int B, int ns,
                                                  unsigned long long total, unsigned long long* keys, int* bags) {
  pdl_entry();
  const int bag = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (bag >= B * ns) return;
  const int t = bag % ns;
  const int lo = off[bag], hi = off[bag + 1];
  for (int e = lo + lane; e < hi; e += 32) {
    const long long r = ids[e];
    keys[e] = (r >= 0 && r < rows[t]) ? (unsigned long long)(rbase[t] + r) : total;
    bags[e] = bag;
  }
}

// Backward, step 3: run heads of the sorted keys (position 0 or a key change), compacted by CUB select.
__global__ void __launch_bounds__(256) emb_heads_k(const unsigned long long* __restrict__ keys, long long nnz,
                                                   unsigned char* head) {
  pdl_entry();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// Backward, step 4 (persistent, warp = run of equal rows, grid-strided over the *nruns runs): the run's dX0
// tokens summed in the sorted (= sample) order, FP_U rows in flight, then E[row] -= lr * sum.  The table row
// is fetched with the run's first rows, so a run of one occurrence costs one round of loads; 64 registers a
// thread keep 32 warps an SM resident (the kernel is latency-bound on short runs).
constexpr int FP_U = 4;
template <typename GT>
__global__ void __launch_bounds__(256, 4) emb_runs_k(const unsigned long long* __restrict__ keys, const int* __restrict__ bags,
                                                     const int* __restrict__ heads, const int* __restrict__ nruns,
                                                     long long nnz, unsigned long long total, const GT* __restrict__ dx0,
                                                     int ns, int nd, int d, int m0, float lr, float* tab) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int nr = *nruns;
  const int nc = (d + 127) >> 7;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < nr; r += gridDim.x * 8) {
    const long long lo = heads[r], hi = r + 1 < nr ? heads[r + 1] : nnz;
    const unsigned long long K = keys[lo];
    if (K >= total) continue;   // the sentinel run of skipped ids
    float* row = tab + (long long)K * d;
    for (int q0 = 0; q0 < nc; q0 += 2) {   // 256 columns per round (d <= 512: at most two rounds)
      float4 w[2], acc[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = 128 * (q0 + q) + 4 * lane;
        w[q] = (q0 + q < nc && col < d) ? *reinterpret_cast<const float4*>(row + col) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (long long p0 = lo; p0 < hi; p0 += FP_U) {
        float4 v[FP_U][2];
#pragma unroll
        for (int u = 0; u < FP_U; ++u) {
          const bool ok = p0 + u < hi;
          const int bag = ok ? bags[p0 + u] : 0;
          const int b = bag / ns, t = bag - b * ns;
          const GT* g = dx0 + ((long long)b * m0 + nd + t) * d;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int col = 128 * (q0 + q) + 4 * lane;
            v[u][q] = (ok && q0 + q < nc && col < d) ? ld4<GT>(g + col) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < FP_U; ++u)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            acc[q].x += v[u][q].x; acc[q].y += v[u][q].y; acc[q].z += v[u][q].z; acc[q].w += v[u][q].w;
          }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = 128 * (q0 + q) + 4 * lane;
        if (q0 + q < nc && col < d) {
          w[q].x -= lr * acc[q].x; w[q].y -= lr * acc[q].y; w[q].z -= lr * acc[q].z; w[q].w -= lr * acc[q].w;
          *reinterpret_cast<float4*>(row + col) = w[q];
        }
      }
    }
  }
}

// dZ_L = dX0[:, :n_dtok] (.) (X0[:, :n_dtok] > 0): the last bottom-MLP layer's ReLU derivative from its stored output
template <typename T>
__global__ void relu_mask_k(const T* __restrict__ dx0, const T* __restrict__ x0, int B, int w, int64_t ld, T* out) {
  pdl_entry();
  const int64_t n = (int64_t)B * w;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / w, j = i - b * w;
    const float g = (float)dx0[b * ld + j], y = (float)x0[b * ld + j];
    out[i] = (T)(y > 0.f ? g : 0.f);
  }
}

}  // namespace

struct dhen_fp {
  int ns, n_dense, nd, d, dt, L, max_B;
  long long max_nnz, total_rows;
  std::vector<long long> rows, rbase;
  std::vector<int> dims;
  float* tables = nullptr;
  long long* d_rbase = nullptr;
  long long* d_rows = nullptr;
  std::vector<float*> Wm, bm, gW, gb;
  std::vector<void*> Wc, bc, H;
  void* dZ[2] = {nullptr, nullptr};
  unsigned long long *keys_in = nullptr, *keys_out = nullptr;
  int *bags_in = nullptr, *bags_out = nullptr, *bad = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int key_bits = 1;
  unsigned char* head = nullptr;   // run-head flags of the sorted keys [nnz]
  int* heads = nullptr;            // compacted run-head positions [nnz]
  int* nruns = nullptr;
  void* sel_tmp = nullptr;
  size_t sel_bytes = 0;
  float* scratch = nullptr;
  size_t scratch_bytes = 0;
  Workspace ws;
  std::vector<void*> allocs;
  // the last forward (referenced, not copied)
  const int* ids = nullptr;
  const int* off = nullptr;
  const void* dense = nullptr;
  void* x0 = nullptr;
  int B = 0;
  long long nnz = 0;
  bool fwd_done = false;
};

namespace {
template <typename P> cudaError_t falloc(dhen_fp* f, P** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e == cudaSuccess) { f->allocs.push_back(q); *p = (P*)q; }
  return e;
}
int64_t numel_of(const dhen_fp* f, int which) {
  if (which < f->ns) return f->rows[which] * f->d;
  const int k = (which - f->ns) / 2;
  return (which - f->ns) % 2 == 0 ? (int64_t)f->dims[k + 1] * f->dims[k] : f->dims[k + 1];
}
dhen_status validate(const dhen_fp_config* c) {
  if (!c) return ffail(DHEN_E_CONFIG, "dhen_fp: config is NULL");
  if (c->n_sparse < 0 || c->n_dense < 0 || c->n_dtok < 0 || c->n_sparse + c->n_dtok <= 0)
    return ffail(DHEN_E_CONFIG, "dhen_fp: need n_sparse + n_dtok > 0 (n_sparse %d, n_dtok %d)", c->n_sparse, c->n_dtok);
  if (c->n_dtok > 0 && c->n_dense <= 0) return ffail(DHEN_E_CONFIG, "dhen_fp: dense tokens need n_dense > 0");
  if (c->d <= 0 || c->d % 4 || c->d > 512) return ffail(DHEN_E_CONFIG, "dhen_fp: d = %d (4 | d, d <= 512)", c->d);
  if (c->dtype != DHEN_FP32 && c->dtype != DHEN_BF16) return ffail(DHEN_E_CONFIG, "dhen_fp: dtype %d", c->dtype);
  if (c->max_batch <= 0 || c->max_nnz < 0) return ffail(DHEN_E_CONFIG, "dhen_fp: max_batch %d max_nnz %lld", c->max_batch, c->max_nnz);
  if (c->n_hidden < 0 || (c->n_hidden > 0 && !c->hidden) || (c->n_sparse > 0 && !c->rows))
    return ffail(DHEN_E_CONFIG, "dhen_fp: hidden / rows arrays missing");
  for (int i = 0; i < c->n_hidden; ++i)
    if (c->hidden[i] <= 0) return ffail(DHEN_E_CONFIG, "dhen_fp: hidden[%d] = %d", i, c->hidden[i]);
  for (int t = 0; t < c->n_sparse; ++t)
    if (c->rows[t] <= 0) return ffail(DHEN_E_CONFIG, "dhen_fp: rows[%d] = %lld", t, c->rows[t]);
  return DHEN_OK;
}
}  // namespace

extern "C" {

long long dhen_fp_param_numel(const dhen_fp_config* c, int which) {
  if (validate(c) != DHEN_OK) return -1;
  const int L = c->n_dtok > 0 ? c->n_hidden + 1 : 0;
  if (which < 0 || which >= c->n_sparse + 2 * L) return -1;
  if (which < c->n_sparse) return c->rows[which] * (long long)c->d;
  std::vector<int> dims;
  dims.push_back(c->n_dense);
  for (int i = 0; i < c->n_hidden; ++i) dims.push_back(c->hidden[i]);
  dims.push_back(c->n_dtok * c->d);
  const int k = (which - c->n_sparse) / 2;
  return (which - c->n_sparse) % 2 == 0 ? (long long)dims[k + 1] * dims[k] : dims[k + 1];
}

void dhen_fp_destroy(dhen_fp* f) {
  if (!f) return;
  for (void* p : f->allocs) cudaFree(p);
  delete f;
}

dhen_status dhen_fp_init(const dhen_fp_config* c, void* stream, dhen_fp** out) {
  if (!out) return ffail(DHEN_E_CONFIG, "dhen_fp_init: out is NULL");
  *out = nullptr;
  const dhen_status v = validate(c);
  if (v != DHEN_OK) return v;
  cudaStream_t st = (cudaStream_t)stream;
  dhen_fp* f = new dhen_fp();
  auto bail = [&](dhen_status s) { dhen_fp_destroy(f); return s; };
#define FA(call)                                                                                        \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) return bail(ffail(e_ == cudaErrorMemoryAllocation ? DHEN_E_NOMEM : DHEN_E_CUDA, \
                                             "dhen_fp_init: %s: %s", #call, cudaGetErrorString(e_)));   \
  } while (0)
  f->ns = c->n_sparse; f->n_dense = c->n_dense; f->nd = c->n_dtok; f->d = c->d; f->dt = c->dtype;
  f->max_B = c->max_batch; f->max_nnz = c->max_nnz;
  f->L = c->n_dtok > 0 ? c->n_hidden + 1 : 0;
  f->total_rows = 0;
  for (int t = 0; t < f->ns; ++t) { f->rows.push_back(c->rows[t]); f->rbase.push_back(f->total_rows); f->total_rows += c->rows[t]; }
  if (f->L) {
    f->dims.push_back(c->n_dense);
    for (int i = 0; i < c->n_hidden; ++i) f->dims.push_back(c->hidden[i]);
    f->dims.push_back(c->n_dtok * c->d);
  }
  const int es = f->dt == DHEN_BF16 ? 2 : 4;
  FA(falloc(f, &f->tables, (size_t)f->total_rows * f->d * 4));
  FA(falloc(f, &f->d_rbase, sizeof(long long) * std::max(1, f->ns)));
  FA(falloc(f, &f->d_rows, sizeof(long long) * std::max(1, f->ns)));
  FA(falloc(f, &f->bad, sizeof(int)));
  if (f->ns) {
    FA(cudaMemcpyAsync(f->d_rbase, f->rbase.data(), sizeof(long long) * f->ns, cudaMemcpyHostToDevice, st));
    FA(cudaMemcpyAsync(f->d_rows, f->rows.data(), sizeof(long long) * f->ns, cudaMemcpyHostToDevice, st));
  }
  FA(cudaMemsetAsync(f->bad, 0, sizeof(int), st));
  // parameters: tables U(+-sqrt(1/R_t)), W_k / b_k U(+-1/sqrt(fan_in)) (R33), one counter stream per tensor
  for (int t = 0; t < f->ns; ++t)
    FA(init_uniform(f->tables + f->rbase[t] * f->d, f->rows[t] * f->d, (float)std::sqrt(1.0 / (double)f->rows[t]),
                    c->seed, 1000 + t, 0, st));
  int wmax = 1;
  for (int k = 0; k < f->L; ++k) {
    const int64_t nw = (int64_t)f->dims[k + 1] * f->dims[k], nb = f->dims[k + 1];
    float *wm, *bm, *gw, *gb;
    void *wc, *bc;
    FA(falloc(f, &wm, nw * 4)); FA(falloc(f, &bm, nb * 4)); FA(falloc(f, &gw, nw * 4)); FA(falloc(f, &gb, nb * 4));
    FA(falloc(f, &wc, nw * es)); FA(falloc(f, &bc, nb * es));
    const float bound = (float)(1.0 / std::sqrt((double)f->dims[k]));
    FA(init_uniform(wm, nw, bound, c->seed, 2 * k, 0, st));
    FA(init_uniform(bm, nb, bound, c->seed, 2 * k + 1, 0, st));
    FA(cast(wm, F32, wc, f->dt, nw, st));
    FA(cast(bm, F32, bc, f->dt, nb, st));
    f->Wm.push_back(wm); f->bm.push_back(bm); f->gW.push_back(gw); f->gb.push_back(gb);
    f->Wc.push_back(wc); f->bc.push_back(bc);
    wmax = std::max(wmax, std::max(f->dims[k], f->dims[k + 1]));
    if (k + 1 < f->L) {
      void* h;
      FA(falloc(f, &h, (size_t)f->max_B * f->dims[k + 1] * es));
      f->H.push_back(h);
    }
  }
  if (f->L) {
    FA(falloc(f, &f->dZ[0], (size_t)f->max_B * wmax * es));
    FA(falloc(f, &f->dZ[1], (size_t)f->max_B * wmax * es));
    f->scratch_bytes = (size_t)4 << 20;
    FA(falloc(f, &f->scratch, f->scratch_bytes));
    f->ws.bytes = (size_t)64 << 20;
    FA(falloc(f, &f->ws.ptr, f->ws.bytes));
  }
  if (f->ns && f->max_nnz > 0) {
    const size_t n = (size_t)f->max_nnz;
    FA(falloc(f, &f->keys_in, n * 8)); FA(falloc(f, &f->keys_out, n * 8));
    FA(falloc(f, &f->bags_in, n * 4)); FA(falloc(f, &f->bags_out, n * 4));
    while (f->key_bits < 64 && (1ull << f->key_bits) <= (unsigned long long)f->total_rows) ++f->key_bits;
    FA(cub::DeviceRadixSort::SortPairs(nullptr, f->cub_bytes, f->keys_in, f->keys_out, f->bags_in, f->bags_out,
                                       (int64_t)n, 0, f->key_bits, st));
    FA(falloc(f, &f->cub_tmp, f->cub_bytes));
    FA(falloc(f, &f->head, n)); FA(falloc(f, &f->heads, n * 4)); FA(falloc(f, &f->nruns, 4));
    FA(cub::DeviceSelect::Flagged(nullptr, f->sel_bytes, cub::CountingInputIterator<int>(0), f->head, f->heads, f->nruns,
                                  (int64_t)n, st));
    FA(falloc(f, &f->sel_tmp, f->sel_bytes));
  }
  FA(cudaStreamSynchronize(st));
#undef FA
  *out = f;
  return DHEN_OK;
}

dhen_status dhen_fp_forward(dhen_fp* f, const int* ids, const int* offsets, long long nnz, const void* dense, int B,
                            void* x0, void* stream) {
  if (!f) return ffail(DHEN_E_STATE, "dhen_fp_forward: fp is NULL");
  if (B <= 0 || B > f->max_B) return ffail(DHEN_E_SHAPE, "dhen_fp_forward: B = %d (max %d)", B, f->max_B);
  if (nnz < 0 || nnz > f->max_nnz) return ffail(DHEN_E_SHAPE, "dhen_fp_forward: nnz = %lld (max %lld)", nnz, f->max_nnz);
  if (!x0 || (f->ns && (!ids || !offsets)) || (f->L && !dense)) return ffail(DHEN_E_ALIGN, "dhen_fp_forward: NULL buffer");
  if (((uintptr_t)x0 % 16) || (dense && (uintptr_t)dense % 16)) return ffail(DHEN_E_ALIGN, "dhen_fp_forward: x0 / dense not 16-B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int m0 = f->nd + f->ns, d = f->d;
  // bottom MLP: H_k = relu(H_{k-1} W_k^T + b_k); the last layer straight into X0's first n_dtok tokens
  for (int k = 0; k < f->L; ++k) {
    const int in = f->dims[k], outw = f->dims[k + 1];
    const void* A = k == 0 ? dense : f->H[k - 1];
    const bool last = k + 1 == f->L;
    Gemm g;
    g.M = B; g.N = outw; g.K = in; g.batch = 1;
    g.a = operand(A, f->dt, in, 1);
    g.b = operand(f->Wc[k], f->dt, in, 1);
    g.c = last ? view(x0, f->dt, (int64_t)m0 * d, 1) : view(f->H[k], f->dt, outw, 1);
    g.e.bias = f->bc[k]; g.e.bias_dt = f->dt; g.e.relu = 1;
    FCK(gemm_run(g, f->ws, st));
  }
  if (f->ns) {
    const int bags = B * f->ns;
    if (f->dt == DHEN_BF16)
      FCK(pdl_launch(emb_fwd_k<__nv_bfloat16>, (bags + 7) / 8, 256, 0, st, f->tables, f->d_rbase, f->d_rows, ids, offsets,
                     B, f->ns, f->nd, d, m0, (__nv_bfloat16*)x0, f->bad));
    else
      FCK(pdl_launch(emb_fwd_k<float>, (bags + 7) / 8, 256, 0, st, f->tables, f->d_rbase, f->d_rows, ids, offsets, B,
                     f->ns, f->nd, d, m0, (float*)x0, f->bad));
    ++g_launches;
  }
  f->ids = ids; f->off = offsets; f->nnz = nnz; f->dense = dense; f->x0 = x0; f->B = B;
  f->fwd_done = true;
  return DHEN_OK;
}

dhen_status dhen_fp_backward_sgd(dhen_fp* f, const void* dx0, float lr, void* stream) {
  if (!f) return ffail(DHEN_E_STATE, "dhen_fp_backward_sgd: fp is NULL");
  if (!f->fwd_done) return ffail(DHEN_E_STATE, "dhen_fp_backward_sgd: no preceding dhen_fp_forward");
  if (!dx0 || ((uintptr_t)dx0 % 16)) return ffail(DHEN_E_ALIGN, "dhen_fp_backward_sgd: dx0 NULL or not 16-B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int B = f->B, m0 = f->nd + f->ns, d = f->d;
  const int es = f->dt == DHEN_BF16 ? 2 : 4;
  if (f->L) {
    // dZ_L = dX0[:, :n_dtok] (.) (X0[:, :n_dtok] > 0)
    const int w = f->nd * d;
    const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)B * w + 255) / 256, 148 * 16);
    if (f->dt == DHEN_BF16)
      FCK(pdl_launch(relu_mask_k<__nv_bfloat16>, grid, 256, 0, st, (const __nv_bfloat16*)dx0, (const __nv_bfloat16*)f->x0,
                     B, w, (int64_t)m0 * d, (__nv_bfloat16*)f->dZ[0]));
    else
      FCK(pdl_launch(relu_mask_k<float>, grid, 256, 0, st, (const float*)dx0, (const float*)f->x0, B, w, (int64_t)m0 * d,
                     (float*)f->dZ[0]));
    ++g_launches;
    int cur = 0;
    for (int k = f->L - 1; k >= 0; --k) {
      const int in = f->dims[k], outw = f->dims[k + 1];
      const void* Hp = k == 0 ? f->dense : f->H[k - 1];
      FCK(fill(f->gb[k], outw, 0.f, st));
      FCK(colsum_add(f->dZ[cur], f->dt, B, outw, outw, f->gb[k], f->scratch, f->scratch_bytes, st));
      Gemm gw;   // dW_k = dZ_k^T H_{k-1}  [out][in], K = B
      gw.M = outw; gw.N = in; gw.K = B; gw.batch = 1;
      gw.a = operand(f->dZ[cur], f->dt, 1, outw);
      gw.b = operand(Hp, f->dt, 1, in);
      gw.c = view(f->gW[k], F32, in, 1);
      FCK(gemm_run(gw, f->ws, st));
      if (k > 0) {   // dZ_{k-1} = (dZ_k W_k) (.) (H_{k-1} > 0)
        Gemm gd;
        gd.M = B; gd.N = in; gd.K = outw; gd.batch = 1;
        gd.a = operand(f->dZ[cur], f->dt, outw, 1);
        gd.b = operand(f->Wc[k], f->dt, 1, in);
        gd.c = view(f->dZ[cur ^ 1], f->dt, in, 1);
        gd.e.mask = view(f->H[k - 1], f->dt, in, 1);
        FCK(gemm_run(gd, f->ws, st));
        cur ^= 1;
      }
    }
    for (int k = 0; k < f->L; ++k) {
      FCK(sgd_cast(f->Wm[k], f->gW[k], lr, f->Wc[k], f->dt, (int64_t)f->dims[k + 1] * f->dims[k], st));
      FCK(sgd_cast(f->bm[k], f->gb[k], lr, f->bc[k], f->dt, f->dims[k + 1], st));
    }
  }
  if (f->ns && f->nnz > 0) {
    const int bags = B * f->ns;
    const unsigned long long total = (unsigned long long)f->total_rows;
    FCK(pdl_launch(emb_keys_k, (bags + 7) / 8, 256, 0, st, f->d_rbase, f->d_rows, f->ids, f->off, B, f->ns, total,
                   f->keys_in, f->bags_in));
    size_t tb = f->cub_bytes;
    FCK(cub::DeviceRadixSort::SortPairs(f->cub_tmp, tb, f->keys_in, f->keys_out, f->bags_in, f->bags_out, (int64_t)f->nnz,
                                        0, f->key_bits, st));
    FCK(pdl_launch(emb_heads_k, 148 * 8, 256, 0, st, f->keys_out, f->nnz, f->head));
    size_t sb = f->sel_bytes;
    FCK(cub::DeviceSelect::Flagged(f->sel_tmp, sb, cub::CountingInputIterator<int>(0), f->head, f->heads, f->nruns,
                                   (int64_t)f->nnz, st));
    if (f->dt == DHEN_BF16)
      FCK(pdl_launch(emb_runs_k<__nv_bfloat16>, 148 * 4, 256, 0, st, f->keys_out, f->bags_out, f->heads, f->nruns, f->nnz,
                     total, (const __nv_bfloat16*)dx0, f->ns, f->nd, d, m0, lr, f->tables));
    else
      FCK(pdl_launch(emb_runs_k<float>, 148 * 4, 256, 0, st, f->keys_out, f->bags_out, f->heads, f->nruns, f->nnz, total,
                     (const float*)dx0, f->ns, f->nd, d, m0, lr, f->tables));
    g_launches += 5;
  }
  (void)es;
  f->fwd_done = false;
  return DHEN_OK;
}

dhen_status dhen_fp_params_io(dhen_fp* f, int which, float* host, int set, void* stream) {
  if (!f || !host) return ffail(DHEN_E_STATE, "dhen_fp_params_io: NULL argument");
  if (which < 0 || which >= f->ns + 2 * f->L) return ffail(DHEN_E_SHAPE, "dhen_fp_params_io: which = %d", which);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = numel_of(f, which);
  float* dev;
  void* copy = nullptr;
  if (which < f->ns) {
    dev = f->tables + f->rbase[which] * f->d;
  } else {
    const int k = (which - f->ns) / 2;
    const bool w = (which - f->ns) % 2 == 0;
    dev = w ? f->Wm[k] : f->bm[k];
    copy = w ? f->Wc[k] : f->bc[k];
  }
  if (set) {
    FCK(cudaMemcpyAsync(dev, host, n * 4, cudaMemcpyHostToDevice, st));
    if (copy) FCK(cast(dev, F32, copy, f->dt, n, st));
  } else {
    FCK(cudaMemcpyAsync(host, dev, n * 4, cudaMemcpyDeviceToHost, st));
  }
  FCK(cudaStreamSynchronize(st));
  return DHEN_OK;
}

long long dhen_fp_bad_ids(dhen_fp* f) {
  if (!f) return -1;
  int h = 0;
  if (cudaMemcpy(&h, f->bad, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return h;
}

}  // extern "C"
