// gemm_simt.cu — exact-FP32-FMA tiled GEMM over strided views (the fp32 mode,
// never TF32) and the fallback for shapes the tcgen05 path does not
// take.  64x64x16 tiles, 256 threads, 4x4 outputs per thread, deterministic
// split-K (fixed-order second pass) for long reductions.
#include "gemm.h"
#include "gemm_epi.cuh"
#include <algorithm>

namespace dhen {

unsigned long long g_launches = 0;

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(Gemm g, int splits, int kchunk, float* ws, int zbase) {
  pdl_entry();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int zb = zbase + blockIdx.z / splits, sp = blockIdx.z % splits;
  const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
  const int kbeg = sp * kchunk;
  const int kend = min(g.K, kbeg + kchunk);
  const T* A = static_cast<const T*>(g.a.ptr);
  const T* Bp = static_cast<const T*>(g.b.ptr);
  const bool a_kc = (g.a.s_k == 1);   // k contiguous in A
  const bool b_kc = (g.b.s_k == 1);
  const int tx = tid % 16, ty = tid / 16;
  float acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;

  for (int k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int e = tid + 256 * q;
      int ii, kk;
      if (a_kc) { ii = e / BK; kk = e % BK; } else { kk = e / BM; ii = e % BM; }
      int gi = i0 + ii, gk = k0 + kk;
      float v = 0.f;
      if (gi < g.M && gk < kend) v = tof<T>(A[g.a.off(zb, gi, gk)]);
      As[kk][ii] = v;
      int jj;
      if (b_kc) { jj = e / BK; kk = e % BK; } else { kk = e / BN; jj = e % BN; }
      int gj = j0 + jj;
      gk = k0 + kk;
      v = 0.f;
      if (gj < g.N && gk < kend) v = tof<T>(Bp[g.b.off(zb, gj, gk)]);
      Bs[kk][jj] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int i = i0 + ty * 4 + r, j = j0 + tx * 4 + c;
      if (i < g.M && j < g.N) {
        if (splits == 1) epi_apply(g, zb, i, j, acc[r][c]);
        else ws[((int64_t)(zb * splits + sp) * g.M + i) * g.N + j] = acc[r][c];
      }
    }
}

// Split-K reduction: block = 32 consecutive output elements (tx) x 8 split lanes (ty); split lane ty
// sums splits ty, ty+8, ... (two independent chains), then the 8 lane sums are combined in fixed order
// -> deterministic, and ~splits/8 dependent loads per thread instead of splits.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(Gemm g, int splits, const float* ws) {
  pdl_entry();
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t mn = (int64_t)g.M * g.N;
  const int64_t total = (int64_t)g.batch * mn;
  for (int64_t e0 = (int64_t)blockIdx.x * 32; e0 < total; e0 += (int64_t)gridDim.x * 32) {
    const int64_t e = e0 + tx;
    float s0 = 0.f, s1 = 0.f;
    if (e < total) {
      const int64_t zb = e / mn, r = e % mn;
      const float* base = ws + zb * splits * mn + r;
      int sp = ty;
      for (; sp + 8 < splits; sp += 16) { s0 += base[(int64_t)sp * mn]; s1 += base[(int64_t)(sp + 8) * mn]; }
      if (sp < splits) s0 += base[(int64_t)sp * mn];
    }
    red[ty][tx] = s0 + s1;
    __syncthreads();
    if (ty == 0 && e < total) {
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) v += red[k][tx];
      const int64_t zb = e / mn, r = e % mn;
      epi_apply(g, (int)zb, (int)(r / g.N), (int)(r % g.N), v);
    }
    __syncthreads();
  }
}

// Split-K reduction for many output elements and few splits: one thread per element, the splits added in
// index order (deterministic), then the fused epilogue.
__global__ void __launch_bounds__(256) splitk_reduce_elem_kernel(Gemm g, int splits, const float* ws) {
  pdl_entry();
  const int64_t mn = (int64_t)g.M * g.N;
  const int64_t total = (int64_t)g.batch * mn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t zb = e / mn, r = e - zb * mn;
    const float* base = ws + zb * splits * mn + r;
    float v = 0.f;
    for (int sp = 0; sp < splits; ++sp) v += __ldcs(base + (int64_t)sp * mn);
    epi_apply(g, (int)zb, (int)(r / g.N), (int)(r % g.N), v);
  }
}

cudaError_t gemm_simt(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.e.ln_gamma || g.e.bits_mode || g.e.bsum || g.e.csum) return cudaErrorNotSupported;   // tcgen05-path-only epilogues
  int tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
  int64_t tiles = (int64_t)tm * tn * g.batch;
  int splits = 1;
  if (g.K > 512 && tiles < 2 * 148) {
    splits = (int)std::min<int64_t>((2 * 148 + tiles - 1) / tiles, (g.K + 255) / 256);
    int64_t need = (int64_t)splits * g.batch * g.M * g.N * 4;
    while (splits > 1 && need > (int64_t)ws.bytes) {
      --splits;
      need = (int64_t)splits * g.batch * g.M * g.N * 4;
    }
  }
  int kchunk = (g.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  if (g.K <= 0) kchunk = 0;
  const int zmax = 65535 / splits;
  for (int zb = 0; zb < g.batch; zb += zmax) {
    int nz = std::min(zmax, g.batch - zb);
    dim3 grid(tn, tm, nz * splits);
    if (g.a.dt == F32)
      pdl_launch(gemm_simt_kernel<float>, grid, 256, 0, st, g, splits, kchunk, ws.ptr, zb);
    else
      pdl_launch(gemm_simt_kernel<__nv_bfloat16>, grid, 256, 0, st, g, splits, kchunk, ws.ptr, zb);
    ++g_launches;
  }
  if (splits > 1) return splitk_reduce(g, splits, ws.ptr, st);
  return cudaGetLastError();
}

cudaError_t splitk_reduce(const Gemm& g, int splits, const float* ws, cudaStream_t st) {
  int64_t total = (int64_t)g.batch * g.M * g.N;
  if (total >= (int64_t)148 * 256 && splits <= 32) {   // enough elements to fill the machine one per thread
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    pdl_launch(splitk_reduce_elem_kernel, blocks, 256, 0, st, g, splits, ws);
    ++g_launches;
    return cudaGetLastError();
  }
  int blocks = (int)std::min<int64_t>((total + 31) / 32, 148 * 8);
  pdl_launch(splitk_reduce_kernel, blocks, 256, 0, st, g, splits, ws);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace dhen
