// fp.cu — NEXT#4: the feature processing layer in front of the DHEN stack ("we use the same feature
// processing layer in DLRM"; readings R32-R34, R36 in DESIGN.md §3).
//
//   sparse: X0[b][n_dtok + t] = sum_{e in bag(b, t)} E_t[ids[e]]          (one pooled token per table)
//   dense:  H_0 = dense, H_k = relu(H_{k-1} W_k^T + b_k), X0[b][0 .. n_dtok) = H_L[b] as n_dtok d-vectors
//   backward + SGD: E_t[r] -= lr sum_{occurrences of r} dX0[b][n_dtok + t]; the bottom MLP by GEMMs + SGD.
//
// Tables are stored as column SHARDS ("slice oversized embedding tables into equal column shards", placed
// by LPT): on one GPU every table is one shard of d columns; with world > 1 each table is cut into S_t equal
// shards and every rank stores only the shards the plan gives it (`plan`).  A shard is a row-major fp32 [R_t][w]
// block.  Forward: one warp per (sample, shard) bag, lanes across the shard's columns (16 B each), four looked-up
// rows in flight, summed in list order; the pooled row goes to X0 (one GPU) or to this rank's send block of the
// pooled all-to-all (world > 1: the rank pools its shards for all world x B samples; after the all-to-all every
// rank assembles its own samples' X0 tokens from every rank's block).  Backward: the reverse all-to-all brings each
// shard owner dX0's columns of its shards for all world x B samples; the occurrence keys (table, row) and their
// bag ids are sorted once (CUB radix sort: stable, so equal rows keep sample order), the run heads compacted by
// CUB select, and a persistent kernel gives each run of equal rows to one warp, which -- for each of this rank's
// shards of that table -- sums the run's gradient rows in that order (four in flight, the table row fetched with
// the first rows) and applies E[row] -= lr * sum in place: deterministic, no atomics, no dense gradient table.
// The bottom MLP runs on the library's tcgen05 GEMM engine (bias + ReLU epilogues, the last layer written straight
// into X0's dense tokens; ReLU-mask epilogues in the backward) and, with world > 1, is data parallel: its
// gradients are all-reduced (sum, rank order) before SGD.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dhen.h"
#include "comm.h"
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

// One column shard of a table.
struct Shard {
  long long base;   // float offset of its [rows][width] block in this rank's shard storage (owned shards)
  long long rows;   // R_t
  int width;        // columns (multiple of 4, <= 512)
  int col0;         // first table column
  int tab;          // table t
  int jt;           // t's index among the tables this rank owns a shard of (the id bags' second index)
  int out;          // column offset of the shard's values in an output / gradient row
};

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

// Forward gather: warp = bag (b, shard j) of nb samples; lane owns columns 4 lane + 128 c (c < NC) of the shard;
// four rows in flight, summed in list order; the pooled row -> out[b * pitch + shard.out ..].  Ids outside
// [0, R_t) are skipped and counted in *bad (once per table: at its first column shard).  NC = 2 when every shard
// is at most 256 columns wide (half the registers: 32 warps an SM in flight; C4 bench shape 3.83 -> 2.83 ms,
// same-box A/B; 48 or 64 warps measured slower), else 4.
template <typename OT, int NC>
__global__ void __launch_bounds__(256, NC == 2 ? 4 : 1) emb_fwd_k(const float* __restrict__ tab, const Shard* __restrict__ sh, int nsh,
                                                 const int* __restrict__ ids, const int* __restrict__ off, int ntab, int nb,
                                                 OT* __restrict__ out, long long pitch, int* bad) {
  pdl_entry();
  const int bag = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (bag >= nb * nsh) return;
  const int b = bag / nsh, j = bag - b * nsh;
  const Shard s = sh[j];
  const int lo = off[b * ntab + s.jt], hi = off[b * ntab + s.jt + 1];
  const float* T = tab + s.base;
  const int w = s.width, nc = (w + 127) >> 7;
  float4 acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int e = lo; e < hi; e += 4) {
    long long r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = e + u < hi ? (long long)__ldg(ids + e + u) : -1;
      if (e + u < hi && (r[u] < 0 || r[u] >= s.rows)) {
        if (lane == 0 && s.col0 == 0) atomicAdd(bad, 1);
        r[u] = -1;
      }
    }
    float4 v[4][NC];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int col = 128 * c + 4 * lane;
        v[u][c] = (r[u] >= 0 && c < nc && col < w) ? __ldg(reinterpret_cast<const float4*>(T + r[u] * w + col))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        acc[c].x += v[u][c].x; acc[c].y += v[u][c].y; acc[c].z += v[u][c].z; acc[c].w += v[u][c].w;
      }
  }
  OT* dst = out + (long long)b * pitch + s.out;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = 128 * c + 4 * lane;
    if (c < nc && col < w) st4<OT>(dst + col, acc[c]);
  }
}

// World > 1: move shard columns between the all-to-all blocks ([rank][B][cmax]) and X0 [B][m0][d]; one warp per
// (sample, global shard).  to_x0: blocks -> X0 (forward assembly), else X0 (dX0) -> blocks (backward).
template <typename T>
__global__ void __launch_bounds__(256) fp_route_k(const Shard* __restrict__ gsh, const int* __restrict__ owner, int ngsh,
                                                  int B, long long cmax, int m0, int nd, int d, T* blocks, T* x0, int to_x0) {
  pdl_entry();
  const int item = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (item >= B * ngsh) return;
  const int b = item / ngsh, g = item - b * ngsh;
  const Shard s = gsh[g];
  T* blk = blocks + ((long long)owner[g] * B + b) * cmax + s.out;
  T* xr = x0 + ((long long)b * m0 + nd + s.tab) * d + s.col0;
  for (int c = lane; c < s.width; c += 32) {
    if (to_x0) xr[c] = blk[c];
    else blk[c] = xr[c];
  }
}

// Backward, step 1: the occurrence keys (owned table jt << 40 | row; skipped ids -> all ones, sorted last) and their
// samples b (the bag is b * ntab + jt), in list order.
__global__ void __launch_bounds__(256) emb_keys_k(const long long* __restrict__ trows, const int* __restrict__ ids,
                                                  const int* __restrict__ off, int ntab, int nb, unsigned long long* keys,
                                                  int* samp) {
  pdl_entry();
  const int bag = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (bag >= nb * ntab) return;
  const int jt = bag % ntab;
  const int lo = off[bag], hi = off[bag + 1];
  const long long R = trows[jt];
  for (int e = lo + lane; e < hi; e += 32) {
    const long long r = ids[e];
    keys[e] = (r >= 0 && r < R) ? (((unsigned long long)jt << 40) | (unsigned long long)r) : ~0ull;
    samp[e] = bag / ntab;
  }
}

// Backward, step 2: run heads of the sorted keys (position 0 or a key change), compacted by CUB select.
__global__ void __launch_bounds__(256) emb_heads_k(const unsigned long long* __restrict__ keys, long long n,
                                                   unsigned char* head) {
  pdl_entry();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// Backward, step 3 (persistent, warp = run of equal rows, grid-strided over the *nruns runs): for each of this
// rank's shards of the run's table, the run's gradient rows (grad[b * pitch + shard.out ..]) summed in the sorted
// (= sample) order, two rows in flight, then E[row] -= lr * sum.  The table row is fetched with the run's first
// rows, so a run of one occurrence costs one round of loads.  The kernel is latency-bound on short runs (three
// occurrences a run on average at the bench shape), so resident warps are what count: 40 registers a thread keep
// 48 warps an SM (measured, C4 bench shape: 11.7 ms at 4 rows in flight x 32 warps, 7.8 ms here; batching 32
// runs' metadata per warp clumps the hot rows of a table onto one warp and was slower).
constexpr int FP_U = 2;
template <typename GT>
__global__ void __launch_bounds__(256, 6) emb_runs_k(const unsigned long long* __restrict__ keys, const int* __restrict__ samp,
                                                     const int* __restrict__ heads, const int* __restrict__ nruns,
                                                     int n, const Shard* __restrict__ sh, const int2* __restrict__ trange,
                                                     int ntab, const GT* __restrict__ grad, long long pitch, float lr,
                                                     float* tab) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int nr = *nruns;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < nr; r += gridDim.x * 8) {
    const int lo = heads[r], hi = r + 1 < nr ? heads[r + 1] : n;
    const unsigned long long K = keys[lo];
    const int jt = (int)(K >> 40);
    if (jt >= ntab) continue;   // the run of skipped ids
    const long long row_i = (long long)(K & ((1ull << 40) - 1));
    const int2 tr = trange[jt];   // this rank's shards of the table: [tr.x, tr.x + tr.y)
    for (int j = tr.x; j < tr.x + tr.y; ++j) {
      const int w = sh[j].width;
      float* row = tab + sh[j].base + row_i * w + 4 * lane;
      const GT* gcol = grad + sh[j].out + 4 * lane;
      for (int c0 = 0; c0 < w; c0 += 256) {   // 256 columns per round (w <= 512: at most two rounds)
        const bool ok0 = c0 + 4 * lane < w, ok1 = c0 + 128 + 4 * lane < w;
        const float4 wv0 = ok0 ? *reinterpret_cast<const float4*>(row + c0) : z4;
        const float4 wv1 = ok1 ? *reinterpret_cast<const float4*>(row + c0 + 128) : z4;
        float4 acc0 = z4, acc1 = z4;
        for (int p0 = lo; p0 < hi; p0 += FP_U) {
          float4 v[FP_U][2];
#pragma unroll
          for (int u = 0; u < FP_U; ++u) {
            const bool ok = p0 + u < hi;
            const GT* g = gcol + (long long)(ok ? samp[p0 + u] : 0) * pitch + c0;
            v[u][0] = (ok && ok0) ? ld4<GT>(g) : z4;
            v[u][1] = (ok && ok1) ? ld4<GT>(g + 128) : z4;
          }
#pragma unroll
          for (int u = 0; u < FP_U; ++u) {
            acc0.x += v[u][0].x; acc0.y += v[u][0].y; acc0.z += v[u][0].z; acc0.w += v[u][0].w;
            acc1.x += v[u][1].x; acc1.y += v[u][1].y; acc1.z += v[u][1].z; acc1.w += v[u][1].w;
          }
        }
        if (ok0)
          *reinterpret_cast<float4*>(row + c0) =
              make_float4(wv0.x - lr * acc0.x, wv0.y - lr * acc0.y, wv0.z - lr * acc0.z, wv0.w - lr * acc0.w);
        if (ok1)
          *reinterpret_cast<float4*>(row + c0 + 128) =
              make_float4(wv1.x - lr * acc1.x, wv1.y - lr * acc1.y, wv1.z - lr * acc1.z, wv1.w - lr * acc1.w);
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

// The column-shard plan, identical on every rank: S_t = the smallest power of two with R_t d / S_t at most
// half of one rank's share of all table elements (as long as a shard keeps >= 32 columns, a multiple of 4); the
// shards placed by LPT -- largest cost first, each onto the least-loaded rank (ties: lowest rank) -- with
// cost = R_t w (the shard's storage; the pooled bytes its lookups move also scale with w).
void plan(const std::vector<long long>& rows, int d, int world, std::vector<int>* S, std::vector<int>* owner) {
  const int ns = (int)rows.size();
  S->assign(ns, 1);
  owner->clear();
  if (world <= 1) { owner->assign(ns, 0); return; }
  double tot = 0;
  for (long long R : rows) tot += (double)R * d;
  const double cap = tot / world / 2;
  for (int t = 0; t < ns; ++t)
    while ((double)rows[t] * d / (*S)[t] > cap && d / ((*S)[t] * 2) >= 32 && (d / ((*S)[t] * 2)) % 4 == 0) (*S)[t] *= 2;
  struct Job { double cost; int t, s; };
  std::vector<Job> jobs;
  for (int t = 0; t < ns; ++t)
    for (int s = 0; s < (*S)[t]; ++s) jobs.push_back({(double)rows[t] * (d / (*S)[t]), t, s});
  std::stable_sort(jobs.begin(), jobs.end(), [](const Job& a, const Job& b) { return a.cost > b.cost; });
  std::vector<double> load(world, 0.0);
  std::vector<std::vector<int>> own(ns);
  for (int t = 0; t < ns; ++t) own[t].assign((*S)[t], 0);
  for (const Job& j : jobs) {
    const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[r] += j.cost;
    own[j.t][j.s] = r;
  }
  for (int t = 0; t < ns; ++t)
    for (int s = 0; s < (*S)[t]; ++s) owner->push_back(own[t][s]);
}

}  // namespace

struct dhen_fp {
  int ns, n_dense, nd, d, dt, L, max_B;
  long long max_nnz;
  int rank = 0, world = 1;
  Comm* comm = nullptr;
  std::vector<long long> rows;
  std::vector<int> dims;
  // gsh: every shard of every table (plan order: t, s) with its owner; lsh: this rank's shards, in that order
  std::vector<Shard> gsh, lsh;
  std::vector<int> gowner, otabs;   // owner rank of each global shard; the tables this rank owns a shard of
  long long cmax = 0;               // widest rank's pooled columns (the all-to-all block width)
  Shard *d_lsh = nullptr, *d_gsh = nullptr;
  int* d_gowner = nullptr;
  int2* d_trange = nullptr;          // per owned table: its shards' range in lsh
  long long* d_trows = nullptr;      // per owned table: R_t
  float* tables = nullptr;
  std::vector<float*> Wm, bm, gW, gb;
  std::vector<void*> Wc, bc, H;
  void* dZ[2] = {nullptr, nullptr};
  void *send = nullptr, *recv = nullptr;   // world > 1: [world][max_B][cmax] blocks (dtype)
  float* mlp_red = nullptr;                // world > 1: staging of the MLP gradient all-reduce
  unsigned long long *keys_in = nullptr, *keys_out = nullptr;
  int *bags_in = nullptr, *bags_out = nullptr, *bad = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int key_bits = 41;
  unsigned char* head = nullptr;   // run-head flags of the sorted keys [max_nnz]
  int* heads = nullptr;            // compacted run-head positions [max_nnz]
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
  if (c->max_batch <= 0 || c->max_nnz < 0 || c->max_nnz > 2147483647LL)   // int32 offsets / run heads
    return ffail(DHEN_E_CONFIG, "dhen_fp: max_batch %d max_nnz %lld", c->max_batch, c->max_nnz);
  if (c->n_hidden < 0 || (c->n_hidden > 0 && !c->hidden) || (c->n_sparse > 0 && !c->rows))
    return ffail(DHEN_E_CONFIG, "dhen_fp: hidden / rows arrays missing");
  for (int i = 0; i < c->n_hidden; ++i)
    if (c->hidden[i] <= 0) return ffail(DHEN_E_CONFIG, "dhen_fp: hidden[%d] = %d", i, c->hidden[i]);
  for (int t = 0; t < c->n_sparse; ++t)
    if (c->rows[t] <= 0 || c->rows[t] >= (1ll << 40)) return ffail(DHEN_E_CONFIG, "dhen_fp: rows[%d] = %lld", t, c->rows[t]);
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

dhen_status dhen_fp_shard_plan(const dhen_fp_config* c, int world, int* shards, int* owner) {
  const dhen_status v = validate(c);
  if (v != DHEN_OK) return v;
  if (world < 1 || !shards || !owner) return ffail(DHEN_E_CONFIG, "dhen_fp_shard_plan: world %d / NULL output", world);
  std::vector<long long> rows(c->rows, c->rows + c->n_sparse);
  std::vector<int> S, own;
  plan(rows, c->d, world, &S, &own);
  std::copy(S.begin(), S.end(), shards);
  std::copy(own.begin(), own.end(), owner);
  return DHEN_OK;
}

void dhen_fp_destroy(dhen_fp* f) {
  if (!f) return;
  delete f->comm;
  for (void* p : f->allocs) cudaFree(p);
  delete f;
}

int dhen_fp_owned_tables(const dhen_fp* f, int* tables) {
  if (!f) return -1;
  if (tables) std::copy(f->otabs.begin(), f->otabs.end(), tables);
  return (int)f->otabs.size();
}

dhen_status dhen_fp_init_dist(const dhen_fp_config* c, const dhen_dist* dist, void* stream, dhen_fp** out) {
  if (!out) return ffail(DHEN_E_CONFIG, "dhen_fp_init: out is NULL");
  *out = nullptr;
  const dhen_status v = validate(c);
  if (v != DHEN_OK) return v;
  const int world = dist ? dist->world : 1, rank = dist ? dist->rank : 0;
  if (world < 1 || rank < 0 || rank >= world) return ffail(DHEN_E_CONFIG, "dhen_fp_init: rank %d of world %d", rank, world);
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
  f->rank = rank; f->world = world;
  f->L = c->n_dtok > 0 ? c->n_hidden + 1 : 0;
  if (world > 1) {
    std::string err;
    f->comm = comm_create(dist->backend, dist->nccl_id, world, rank, &err);
    if (!f->comm) return bail(ffail(DHEN_E_NCCL, "dhen_fp_init: %s", err.c_str()));
  }
  // ---- the shard plan and this rank's shards
  for (int t = 0; t < f->ns; ++t) f->rows.push_back(c->rows[t]);
  std::vector<int> S, own;
  plan(f->rows, f->d, world, &S, &own);
  std::vector<long long> colsum(world, 0);
  std::vector<int2> trange;
  std::vector<long long> trows;
  long long base = 0;
  for (int t = 0, g = 0; t < f->ns; ++t)
    for (int s = 0; s < S[t]; ++s, ++g) {
      Shard sh;
      sh.rows = f->rows[t]; sh.width = f->d / S[t]; sh.col0 = s * sh.width; sh.tab = t;
      sh.out = (int)colsum[own[g]];   // offset in its owner's all-to-all block (world > 1)
      colsum[own[g]] += sh.width;
      sh.base = 0; sh.jt = 0;
      f->gsh.push_back(sh);
      f->gowner.push_back(own[g]);
      if (own[g] == rank) {
        if (f->otabs.empty() || f->otabs.back() != t) {
          f->otabs.push_back(t);
          trange.push_back(make_int2((int)f->lsh.size(), 0));
          trows.push_back(f->rows[t]);
        }
        ++trange.back().y;
        sh.base = base;
        base += sh.rows * sh.width;
        sh.jt = (int)f->otabs.size() - 1;
        if (world == 1) sh.out = (f->nd + t) * f->d + sh.col0;   // straight into X0's token
        f->lsh.push_back(sh);
      }
    }
  for (long long cs : colsum) f->cmax = std::max(f->cmax, cs);
  const int es = f->dt == DHEN_BF16 ? 2 : 4;
  FA(falloc(f, &f->tables, (size_t)std::max(1ll, base) * 4));
  FA(falloc(f, &f->bad, sizeof(int)));
  FA(cudaMemsetAsync(f->bad, 0, sizeof(int), st));
  FA(falloc(f, &f->d_lsh, sizeof(Shard) * std::max<size_t>(1, f->lsh.size())));
  FA(falloc(f, &f->d_gsh, sizeof(Shard) * std::max<size_t>(1, f->gsh.size())));
  FA(falloc(f, &f->d_gowner, sizeof(int) * std::max<size_t>(1, f->gowner.size())));
  FA(falloc(f, &f->d_trange, sizeof(int2) * std::max<size_t>(1, trange.size())));
  FA(falloc(f, &f->d_trows, sizeof(long long) * std::max<size_t>(1, trows.size())));
  if (!f->lsh.empty()) {
    FA(cudaMemcpyAsync(f->d_lsh, f->lsh.data(), sizeof(Shard) * f->lsh.size(), cudaMemcpyHostToDevice, st));
    FA(cudaMemcpyAsync(f->d_trange, trange.data(), sizeof(int2) * trange.size(), cudaMemcpyHostToDevice, st));
    FA(cudaMemcpyAsync(f->d_trows, trows.data(), sizeof(long long) * trows.size(), cudaMemcpyHostToDevice, st));
  }
  if (!f->gsh.empty()) {
    FA(cudaMemcpyAsync(f->d_gsh, f->gsh.data(), sizeof(Shard) * f->gsh.size(), cudaMemcpyHostToDevice, st));
    FA(cudaMemcpyAsync(f->d_gowner, f->gowner.data(), sizeof(int) * f->gowner.size(), cudaMemcpyHostToDevice, st));
  }
  // ---- parameters: tables U(+-sqrt(1/R_t)) in the full table's element order (one counter stream per table, so
  // every plan holds the same values), W_k / b_k U(+-1/sqrt(fan_in)) (R33)
  {
    float* tmp = nullptr;
    long long rmax = 0;
    for (const Shard& s : f->lsh) rmax = std::max(rmax, s.rows);
    if (!f->lsh.empty() && world > 1) FA(falloc(f, &tmp, (size_t)rmax * f->d * 4));
    int last = -1;
    for (const Shard& s : f->lsh) {
      const float bound = (float)std::sqrt(1.0 / (double)s.rows);
      if (world == 1) {
        FA(init_uniform(f->tables + s.base, s.rows * f->d, bound, c->seed, 1000 + s.tab, 0, st));
        continue;
      }
      if (s.tab != last) FA(init_uniform(tmp, s.rows * f->d, bound, c->seed, 1000 + s.tab, 0, st));
      last = s.tab;
      FA(cudaMemcpy2DAsync(f->tables + s.base, s.width * 4, tmp + s.col0, f->d * 4, s.width * 4, s.rows,
                           cudaMemcpyDeviceToDevice, st));
    }
  }
  if (f->L) {
    f->dims.push_back(c->n_dense);
    for (int i = 0; i < c->n_hidden; ++i) f->dims.push_back(c->hidden[i]);
    f->dims.push_back(c->n_dtok * c->d);
  }
  int wmax = 1;
  long long mlp_n = 0;
  for (int k = 0; k < f->L; ++k) {
    const int64_t nw = (int64_t)f->dims[k + 1] * f->dims[k], nb = f->dims[k + 1];
    mlp_n = std::max<long long>(mlp_n, nw);
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
    if (world > 1) FA(falloc(f, &f->mlp_red, (size_t)mlp_n * 4));
  }
  if (world > 1 && f->ns) {
    const size_t nblk = (size_t)world * f->max_B * f->cmax;
    FA(falloc(f, &f->send, nblk * es));
    FA(falloc(f, &f->recv, nblk * es));
  }
  if (!f->lsh.empty() && f->max_nnz > 0) {
    const size_t n = (size_t)f->max_nnz;
    FA(falloc(f, &f->keys_in, n * 8)); FA(falloc(f, &f->keys_out, n * 8));
    FA(falloc(f, &f->bags_in, n * 4)); FA(falloc(f, &f->bags_out, n * 4));
    f->key_bits = 41;   // (owned table, row); skipped ids are all ones and sort last
    while ((1ull << (f->key_bits - 40)) <= (unsigned long long)f->otabs.size()) ++f->key_bits;
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

dhen_status dhen_fp_init(const dhen_fp_config* c, void* stream, dhen_fp** out) {
  return dhen_fp_init_dist(c, nullptr, stream, out);
}

dhen_status dhen_fp_forward(dhen_fp* f, const int* ids, const int* offsets, long long nnz, const void* dense, int B,
                            void* x0, void* stream) {
  if (!f) return ffail(DHEN_E_STATE, "dhen_fp_forward: fp is NULL");
  if (B <= 0 || B > f->max_B) return ffail(DHEN_E_SHAPE, "dhen_fp_forward: B = %d (max %d)", B, f->max_B);
  if (nnz < 0 || nnz > f->max_nnz) return ffail(DHEN_E_SHAPE, "dhen_fp_forward: nnz = %lld (max %lld)", nnz, f->max_nnz);
  if (!x0 || (!f->otabs.empty() && (!ids || !offsets)) || (f->L && !dense))
    return ffail(DHEN_E_ALIGN, "dhen_fp_forward: NULL buffer");
  if (((uintptr_t)x0 % 16) || (dense && (uintptr_t)dense % 16)) return ffail(DHEN_E_ALIGN, "dhen_fp_forward: x0 / dense not 16-B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int m0 = f->nd + f->ns, d = f->d;
  const bool bf = f->dt == DHEN_BF16;
  // bottom MLP (this rank's samples): H_k = relu(H_{k-1} W_k^T + b_k); the last layer straight into X0's dense tokens
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
  // pooled lookups of this rank's shards: for its own B samples into X0 (one GPU), or for all world x B samples
  // into its send block, then the all-to-all and the assembly of this rank's X0 tokens from every rank's block
  const int nb = f->world * B, nl = (int)f->lsh.size(), nt = (int)f->otabs.size();
  if (nl) {
    const unsigned grid = (unsigned)(((long long)nb * nl + 7) / 8);
    void* dst = f->world == 1 ? x0 : f->send;
    const long long pitch = f->world == 1 ? (long long)m0 * d : f->cmax;
    int wmax = 0;
    for (const Shard& sh_ : f->lsh) wmax = std::max(wmax, sh_.width);
    if (bf && wmax <= 256)
      FCK(pdl_launch(emb_fwd_k<__nv_bfloat16, 2>, grid, 256, 0, st, f->tables, f->d_lsh, nl, ids, offsets, nt, nb,
                     (__nv_bfloat16*)dst, pitch, f->bad));
    else if (bf)
      FCK(pdl_launch(emb_fwd_k<__nv_bfloat16, 4>, grid, 256, 0, st, f->tables, f->d_lsh, nl, ids, offsets, nt, nb,
                     (__nv_bfloat16*)dst, pitch, f->bad));
    else if (wmax <= 256)
      FCK(pdl_launch(emb_fwd_k<float, 2>, grid, 256, 0, st, f->tables, f->d_lsh, nl, ids, offsets, nt, nb, (float*)dst,
                     pitch, f->bad));
    else
      FCK(pdl_launch(emb_fwd_k<float, 4>, grid, 256, 0, st, f->tables, f->d_lsh, nl, ids, offsets, nt, nb, (float*)dst,
                     pitch, f->bad));
    ++g_launches;
  }
  if (f->world > 1 && f->ns) {
    if (f->comm->all_to_all(f->send, f->recv, (size_t)B * f->cmax, bf ? BF16 : F32, st))
      return ffail(DHEN_E_NCCL, "dhen_fp_forward: pooled all-to-all (%s): %s", f->comm->name(), f->comm->err.c_str());
    const int ng = (int)f->gsh.size();
    const unsigned grid = (unsigned)(((long long)B * ng + 7) / 8);
    if (bf)
      FCK(pdl_launch(fp_route_k<__nv_bfloat16>, grid, 256, 0, st, f->d_gsh, f->d_gowner, ng, B, f->cmax, m0, f->nd, d,
                     (__nv_bfloat16*)f->recv, (__nv_bfloat16*)x0, 1));
    else
      FCK(pdl_launch(fp_route_k<float>, grid, 256, 0, st, f->d_gsh, f->d_gowner, ng, B, f->cmax, m0, f->nd, d,
                     (float*)f->recv, (float*)x0, 1));
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
  const bool bf = f->dt == DHEN_BF16;
  // ---- tables: the gradient rows of this rank's shards (dX0 itself, or -- after the reverse all-to-all -- all
  // world x B samples' columns of its shards), then the sorted-run SGD
  const void* grad = dx0;
  long long pitch = (long long)m0 * d;
  if (f->world > 1 && f->ns) {
    const int ng = (int)f->gsh.size();
    const unsigned grid = (unsigned)(((long long)B * ng + 7) / 8);
    if (bf)
      FCK(pdl_launch(fp_route_k<__nv_bfloat16>, grid, 256, 0, st, f->d_gsh, f->d_gowner, ng, B, f->cmax, m0, f->nd, d,
                     (__nv_bfloat16*)f->send, (__nv_bfloat16*)const_cast<void*>(dx0), 0));
    else
      FCK(pdl_launch(fp_route_k<float>, grid, 256, 0, st, f->d_gsh, f->d_gowner, ng, B, f->cmax, m0, f->nd, d,
                     (float*)f->send, (float*)const_cast<void*>(dx0), 0));
    ++g_launches;
    if (f->comm->all_to_all(f->send, f->recv, (size_t)B * f->cmax, bf ? BF16 : F32, st))
      return ffail(DHEN_E_NCCL, "dhen_fp_backward_sgd: gradient all-to-all (%s): %s", f->comm->name(), f->comm->err.c_str());
    grad = f->recv;
    pitch = f->cmax;
  }
  const int nb = f->world * B, nt = (int)f->otabs.size();
  if (nt && f->nnz > 0) {
    const long long n = f->nnz;
    FCK(pdl_launch(emb_keys_k, (unsigned)(((long long)nb * nt + 7) / 8), 256, 0, st, f->d_trows, f->ids, f->off, nt, nb,
                   f->keys_in, f->bags_in));
    size_t tb = f->cub_bytes;
    FCK(cub::DeviceRadixSort::SortPairs(f->cub_tmp, tb, f->keys_in, f->keys_out, f->bags_in, f->bags_out, (int64_t)n, 0,
                                        f->key_bits, st));
    FCK(pdl_launch(emb_heads_k, 148 * 8, 256, 0, st, f->keys_out, n, f->head));
    size_t sb = f->sel_bytes;
    FCK(cub::DeviceSelect::Flagged(f->sel_tmp, sb, cub::CountingInputIterator<int>(0), f->head, f->heads, f->nruns,
                                   (int64_t)n, st));
    if (bf)
      FCK(pdl_launch(emb_runs_k<__nv_bfloat16>, 148 * 6, 256, 0, st, f->keys_out, f->bags_out, f->heads, f->nruns, (int)n,
                     f->d_lsh, f->d_trange, nt, (const __nv_bfloat16*)grad, pitch, lr, f->tables));
    else
      FCK(pdl_launch(emb_runs_k<float>, 148 * 6, 256, 0, st, f->keys_out, f->bags_out, f->heads, f->nruns, (int)n, f->d_lsh,
                     f->d_trange, nt, (const float*)grad, pitch, lr, f->tables));
    g_launches += 5;
  }
  // ---- bottom MLP (this rank's samples; world > 1: gradients all-reduced, rank order, before SGD)
  if (f->L) {
    const int w = f->nd * d;
    const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)B * w + 255) / 256, 148 * 16);
    if (bf)
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
    if (f->world > 1) {   // data-parallel bottom MLP: sum the ranks' gradients (each already carries 1 / B_global)
      for (int k = 0; k < f->L; ++k) {
        const int64_t nw = (int64_t)f->dims[k + 1] * f->dims[k];
        if (f->comm->all_reduce(f->gW[k], f->mlp_red, nw, F32, st))
          return ffail(DHEN_E_NCCL, "dhen_fp_backward_sgd: MLP all-reduce: %s", f->comm->err.c_str());
        FCK(cudaMemcpyAsync(f->gW[k], f->mlp_red, nw * 4, cudaMemcpyDeviceToDevice, st));
        if (f->comm->all_reduce(f->gb[k], f->mlp_red, f->dims[k + 1], F32, st))
          return ffail(DHEN_E_NCCL, "dhen_fp_backward_sgd: MLP all-reduce: %s", f->comm->err.c_str());
        FCK(cudaMemcpyAsync(f->gb[k], f->mlp_red, f->dims[k + 1] * 4, cudaMemcpyDeviceToDevice, st));
      }
    }
    for (int k = 0; k < f->L; ++k) {
      FCK(sgd_cast(f->Wm[k], f->gW[k], lr, f->Wc[k], f->dt, (int64_t)f->dims[k + 1] * f->dims[k], st));
      FCK(sgd_cast(f->bm[k], f->gb[k], lr, f->bc[k], f->dt, f->dims[k + 1], st));
    }
  }
  f->fwd_done = false;
  return DHEN_OK;
}

dhen_status dhen_fp_params_io(dhen_fp* f, int which, float* host, int set, void* stream) {
  if (!f || !host) return ffail(DHEN_E_STATE, "dhen_fp_params_io: NULL argument");
  if (which < 0 || which >= f->ns + 2 * f->L) return ffail(DHEN_E_SHAPE, "dhen_fp_params_io: which = %d", which);
  cudaStream_t st = (cudaStream_t)stream;
  if (which < f->ns) {   // the [R_t][d] table; only this rank's column shards are read / written
    for (const Shard& s : f->lsh) {
      if (s.tab != which) continue;
      if (set)
        FCK(cudaMemcpy2DAsync(f->tables + s.base, s.width * 4, host + s.col0, f->d * 4, s.width * 4, s.rows,
                              cudaMemcpyHostToDevice, st));
      else
        FCK(cudaMemcpy2DAsync(host + s.col0, f->d * 4, f->tables + s.base, s.width * 4, s.width * 4, s.rows,
                              cudaMemcpyDeviceToHost, st));
    }
    FCK(cudaStreamSynchronize(st));
    return DHEN_OK;
  }
  const int64_t n = numel_of(f, which);
  const int k = (which - f->ns) / 2;
  const bool w = (which - f->ns) % 2 == 0;
  float* dev = w ? f->Wm[k] : f->bm[k];
  void* copy = w ? f->Wc[k] : f->bc[k];
  if (set) {
    FCK(cudaMemcpyAsync(dev, host, n * 4, cudaMemcpyHostToDevice, st));
    FCK(cast(dev, F32, copy, f->dt, n, st));
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
