// kernels.cu — memory-bound DHEN kernels: triangle gather/scatter (Dot), LayerNorm
// fwd/bwd, column sums, softmax fwd/bwd, DCN backward elementwise, 3x3 conv,
// head + BCE loss, SGD.  Warp-per-row reductions via shuffles; every cross-block
// reduction is a fixed-order two-pass (deterministic).
#include "kernels.h"
#include "tuning.h"
#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace dhen {

static inline int nblocks(int64_t n, int per = 256, int cap = 148 * 32) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, cap));
}

// ------------------------------------------------------------------ Dot triangle
__global__ void triu_extract_k(const float* G, void* Z, int dt, int B, int m, int64_t ldz) {
  pdl_entry();
  const int h = m * (m - 1) / 2;
  int64_t total = (int64_t)B * h;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(t / h), p = (int)(t % h);
    // invert p(i,j) = i*m - i(i+1)/2 + (j-i-1)
    int i = 0, rem = p;
    while (rem >= m - 1 - i) { rem -= m - 1 - i; ++i; }
    int j = i + 1 + rem;
    st_from_f32(Z, (int64_t)b * ldz + p, dt, G[((int64_t)b * m + i) * m + j]);
  }
}
cudaError_t triu_extract(const float* G, void* Z, int dt, int B, int m, int64_t ldz, cudaStream_t st) {
  int64_t total = (int64_t)B * m * (m - 1) / 2;
  pdl_launch(triu_extract_k, nblocks(total), 256, 0, st, G, Z, dt, B, m, ldz);
  ++g_launches;
  return cudaGetLastError();
}

// One block per sample: the packed triangle (h values, contiguous) is staged in shared memory, then the m x m
// matrix is written row-major with 8-element vector stores (m % 8 == 0) or scalars.
__global__ void __launch_bounds__(256) sym_from_triu_k(const void* dZ, void* S, int dt, int m, int64_t ldz) {
  pdl_entry();
  extern __shared__ float tri[];          // [h] triangle values, then [m] row bases
  const int h = m * (m - 1) / 2;
  int* rb = reinterpret_cast<int*>(tri + h);   // rb[i] + j = index of pair (i, j > i)
  const int b = blockIdx.x;
  if (dt == BF16 && (ldz % 8) == 0 && (h % 8) == 0) {   // 16-B loads of 8 bf16
    const uint4* src = reinterpret_cast<const uint4*>((const __nv_bfloat16*)dZ + (int64_t)b * ldz);
    for (int q = threadIdx.x; q < h / 8; q += blockDim.x) {
      const uint4 u = __ldg(src + q);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) { tri[8 * q + 2 * t] = __uint_as_float(w[t] << 16); tri[8 * q + 2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u); }
    }
  } else {
    for (int p = threadIdx.x; p < h; p += blockDim.x) tri[p] = ld_as_f32(dZ, (int64_t)b * ldz + p, dt);
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) rb[i] = i * m - i * (i + 1) / 2 - i - 1;
  __syncthreads();
  const int64_t base = (int64_t)b * m * m;
  auto val = [&](int i, int j) -> float { return j > i ? tri[rb[i] + j] : (j < i ? tri[rb[j] + i] : 0.f); };
  if (dt == BF16 && (m % 8) == 0) {
    const int cpr = m / 8;
    for (int q = threadIdx.x; q < m * cpr; q += blockDim.x) {
      const int i = q / cpr, j0 = (q - i * cpr) * 8;
      uint32_t w[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(val(i, j0 + 2 * t), val(i, j0 + 2 * t + 1));
        w[t] = *reinterpret_cast<uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>((__nv_bfloat16*)S + base + (int64_t)i * m + j0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    for (int q = threadIdx.x; q < m * m; q += blockDim.x) st_from_f32(S, base + q, dt, val(q / m, q % m));
  }
}
// bf16, m % 8 == 0: one warp per triangle row i scatters its pairs into a dense bf16 m x (m+2) shared image,
// both (i, j) and (j, i); the +2 pad makes the transposed column writes and the 4-byte row reads of the
// store phase conflict-free.  Values are copied, not re-rounded, so the result equals sym_from_triu_k's.
__global__ void __launch_bounds__(256) sym_from_triu_bf16_k(const __nv_bfloat16* __restrict__ dZ,
                                                             __nv_bfloat16* __restrict__ S, int m, int64_t ldz, int stage) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char sym_raw[];
  __nv_bfloat16* D = reinterpret_cast<__nv_bfloat16*>(sym_raw);   // [m][m + 2], then the staged triangle [h]
  const int P = m + 2, b = blockIdx.x, lane = threadIdx.x & 31, nw = blockDim.x >> 5, h = m * (m - 1) / 2;
  const __nv_bfloat16* z = dZ + (int64_t)b * ldz;
  if (stage) {   // all of the triangle in flight at once (16-B loads), then scattered from shared memory
    uint4* t = reinterpret_cast<uint4*>(D + m * P);
    const uint4* src = reinterpret_cast<const uint4*>(z);
    for (int q = threadIdx.x; q < h / 8; q += blockDim.x) t[q] = __ldg(src + q);
    z = D + m * P;
    __syncthreads();
  }
  for (int i = threadIdx.x >> 5; i < m; i += nw) {
    const int rbi = i * m - i * (i + 1) / 2 - i - 1;               // rbi + j = index of pair (i, j > i)
    if (lane == 0) D[i * P + i] = __float2bfloat16(0.f);
    for (int j = i + 1 + lane; j < m; j += 32) {
      const __nv_bfloat16 v = z[rbi + j];   // shared (staged) or global
      D[i * P + j] = v;
      D[j * P + i] = v;
    }
  }
  __syncthreads();
  const int cpr = m / 8;
  const int64_t base = (int64_t)b * m * m;
  for (int q = threadIdx.x; q < m * cpr; q += blockDim.x) {
    const int i = q / cpr, j0 = (q - i * cpr) * 8;
    const uint32_t* r = reinterpret_cast<const uint32_t*>(D + i * P + j0);
    *reinterpret_cast<uint4*>(S + base + (int64_t)i * m + j0) = make_uint4(r[0], r[1], r[2], r[3]);
  }
}
cudaError_t sym_from_triu(const void* dZ, void* S, int dt, int B, int m, int64_t ldz, cudaStream_t st) {
  // dhen_tuning.sym: 0 the staged-triangle kernel; 1 the dense image, triangle staged in shared memory;
  // 2 the dense image read from global.  Default (-1) by measurement (tools/gpu_sym.sh, one B200): dense for
  // m >= 128 (C4 1.60 -> 1.14 ms/step), staged triangle at m = 64 (C2 29.8 vs 32.0 us/step).
  const int mode = tune().sym >= 0 ? tune().sym : (m >= 128 ? 1 : 0);
  const int stage = mode == 1 && (ldz % 8) == 0 && ((m * (m - 1) / 2) % 8) == 0;
  if (mode && dt == BF16 && (m % 8) == 0 && (size_t)m * (m + 2) * 2 + (size_t)m * m <= 200 * 1024) {
    const size_t sm = (size_t)m * (m + 2) * 2 + (stage ? (size_t)m * (m - 1) : 0);
    static size_t attr_d = 48 * 1024;
    if (sm > attr_d) {
      cudaFuncSetAttribute(sym_from_triu_bf16_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr_d = sm;
    }
    pdl_launch(sym_from_triu_bf16_k, B, 256, sm, st, (const __nv_bfloat16*)dZ, (__nv_bfloat16*)S, m, ldz, stage);
    ++g_launches;
    return cudaGetLastError();
  }
  const size_t sm = ((size_t)m * (m - 1) / 2 + m) * sizeof(float);
  if (sm > 200 * 1024) return cudaErrorInvalidValue;
  static size_t attr = 48 * 1024;
  if (sm > attr) {
    cudaFuncSetAttribute(sym_from_triu_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = sm;
  }
  pdl_launch(sym_from_triu_k, B, 256, sm, st, dZ, S, dt, m, ldz);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ vector IO helpers
template <int VEC, typename T> struct VIO;
template <> struct VIO<8, __nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* o) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) { o[2 * t] = __uint_as_float(w[t] << 16); o[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u); }
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float* v) {
    uint4 u;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]),
                   h2 = __floats2bfloat162_rn(v[4], v[5]), h3 = __floats2bfloat162_rn(v[6], v[7]);
    u.x = *reinterpret_cast<uint32_t*>(&h0); u.y = *reinterpret_cast<uint32_t*>(&h1);
    u.z = *reinterpret_cast<uint32_t*>(&h2); u.w = *reinterpret_cast<uint32_t*>(&h3);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct VIO<4, __nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* o) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    o[0] = __uint_as_float(u.x << 16); o[1] = __uint_as_float(u.x & 0xffff0000u);
    o[2] = __uint_as_float(u.y << 16); o[3] = __uint_as_float(u.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float* v) {
    uint2 u;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
    u.x = *reinterpret_cast<uint32_t*>(&h0); u.y = *reinterpret_cast<uint32_t*>(&h1);
    *reinterpret_cast<uint2*>(p) = u;
  }
};
template <> struct VIO<2, __nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* o) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    o[0] = __uint_as_float(u << 16); o[1] = __uint_as_float(u & 0xffff0000u);
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float* v) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[0], v[1]);
    *reinterpret_cast<__nv_bfloat162*>(p) = h;
  }
};
template <> struct VIO<1, __nv_bfloat16> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16* p, float* o) { o[0] = __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, const float* v) { *p = __float2bfloat16_rn(v[0]); }
};
template <int VEC> struct VIO<VEC, float> {
  static __device__ __forceinline__ void ld(const float* p, float* o) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
      for (int t = 0; t < VEC; t += 4) {
        const float4 v = *reinterpret_cast<const float4*>(p + t);
        o[t] = v.x; o[t + 1] = v.y; o[t + 2] = v.z; o[t + 3] = v.w;
      }
    } else if constexpr (VEC == 2) {
      const float2 v = *reinterpret_cast<const float2*>(p);
      o[0] = v.x; o[1] = v.y;
    } else {
      o[0] = *p;
    }
  }
  static __device__ __forceinline__ void st(float* p, const float* v) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
      for (int t = 0; t < VEC; t += 4) *reinterpret_cast<float4*>(p + t) = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
    } else if constexpr (VEC == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
      *p = v[0];
    }
  }
};

// ------------------------------------------------------------------ LayerNorm (vectorised)
// One warp per row of d; lane owns NCH chunks of VEC consecutive elements: element (j*32 + lane)*VEC.
template <typename T, int VEC, int NCH>
__global__ void __launch_bounds__(256) ln_fwd_v(const float* __restrict__ U, const T* __restrict__ addx,
                                                const T* __restrict__ gamma, const T* __restrict__ beta, float eps,
                                                int64_t rows, int d, T* __restrict__ Y, T* __restrict__ Rsave,
                                                float* __restrict__ mu, float* __restrict__ rstd) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    float v[NCH][VEC];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = (j * 32 + lane) * VEC;
      VIO<VEC, float>::ld(U + r * d + c, v[j]);
      if (addx) {
        float x[VEC];
        VIO<VEC, T>::ld(addx + r * d + c, x);
#pragma unroll
        for (int t = 0; t < VEC; ++t) v[j][t] += x[t];
      }
#pragma unroll
      for (int t = 0; t < VEC; ++t) s += v[j][t];
    }
    const float mean = warp_sum(s) / d;
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NCH; ++j)
#pragma unroll
      for (int t = 0; t < VEC; ++t) { const float q = v[j][t] - mean; s2 += q * q; }
    const float rs = rsqrtf(warp_sum(s2) / d + eps);
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = (j * 32 + lane) * VEC;
      float g[VEC], b[VEC], y[VEC];
      VIO<VEC, T>::ld(gamma + c, g);
      VIO<VEC, T>::ld(beta + c, b);
#pragma unroll
      for (int t = 0; t < VEC; ++t) y[t] = (v[j][t] - mean) * rs * g[t] + b[t];
      VIO<VEC, T>::st(Y + r * d + c, y);
      if (Rsave) VIO<VEC, T>::st(Rsave + r * d + c, v[j]);
    }
    if (lane == 0) { mu[r] = mean; rstd[r] = rs; }
  }
}

template <typename TD, typename T, int VEC, int NCH>
__global__ void __launch_bounds__(256) ln_bwd_v(const TD* __restrict__ dY, const T* __restrict__ Rsave,
                                                const float* __restrict__ mu, const float* __restrict__ rstd,
                                                const T* __restrict__ gamma, int64_t rows, int d, T* __restrict__ dR,
                                                float* __restrict__ acc, int acc_mode, float* __restrict__ part,
                                                int64_t rows_per_block) {
  pdl_entry();
  extern __shared__ float sred[];   // [8 warps][2][d]
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  const int64_t r0 = blockIdx.x * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  float pg[NCH][VEC], pb[NCH][VEC], g[NCH][VEC];
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    VIO<VEC, T>::ld(gamma + (j * 32 + lane) * VEC, g[j]);
#pragma unroll
    for (int t = 0; t < VEC; ++t) { pg[j][t] = 0.f; pb[j][t] = 0.f; }
  }
  for (int64_t r = r0 + w; r < r1; r += 8) {
    float xh[NCH][VEC], gy[NCH][VEC];
    float s1 = 0.f, s2 = 0.f;
    const float m_ = mu[r], rs = rstd[r];
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = (j * 32 + lane) * VEC;
      float dy[VEC], x[VEC];
      VIO<VEC, TD>::ld(dY + r * d + c, dy);
      VIO<VEC, T>::ld(Rsave + r * d + c, x);
#pragma unroll
      for (int t = 0; t < VEC; ++t) {
        xh[j][t] = (x[t] - m_) * rs;
        gy[j][t] = dy[t] * g[j][t];
        pg[j][t] += dy[t] * xh[j][t];
        pb[j][t] += dy[t];
        s1 += gy[j][t];
        s2 += gy[j][t] * xh[j][t];
      }
    }
    s1 = warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = (j * 32 + lane) * VEC;
      float o[VEC];
#pragma unroll
      for (int t = 0; t < VEC; ++t) o[t] = rs * (gy[j][t] - s1 - xh[j][t] * s2);
      VIO<VEC, T>::st(dR + r * d + c, o);
      if (acc_mode) {
        float q[VEC];
        VIO<VEC, T>::ld(dR + r * d + c, q);   // the stored (rounded) value feeds the residual path
        if (acc_mode == 2) {
          float a[VEC];
          VIO<VEC, float>::ld(acc + r * d + c, a);
#pragma unroll
          for (int t = 0; t < VEC; ++t) q[t] += a[t];
        }
        VIO<VEC, float>::st(acc + r * d + c, q);
      }
    }
  }
  // block reduction of the dgamma / dbeta partials in fixed warp order
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = (j * 32 + lane) * VEC;
#pragma unroll
    for (int t = 0; t < VEC; ++t) { sred[(w * 2) * d + c + t] = pg[j][t]; sred[(w * 2 + 1) * d + c + t] = pb[j][t]; }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int ww = 0; ww < 8; ++ww) { a += sred[(ww * 2) * d + c]; b += sred[(ww * 2 + 1) * d + c]; }
    part[(int64_t)blockIdx.x * 2 * d + c] = a;
    part[(int64_t)blockIdx.x * 2 * d + d + c] = b;
  }
}

// (VEC, NCH) for a row length d; {0,0} = no vectorised variant (generic kernels)
static inline void ln_shape(int d, int& vec, int& nch) {
  vec = 0; nch = 0;
  if (d % 256 == 0 && d / 256 <= 4) { vec = 8; nch = d / 256; }
  else if (d % 128 == 0 && d / 128 <= 3) { vec = 4; nch = d / 128; }
  else if (d % 64 == 0 && d / 64 <= 3) { vec = 2; nch = d / 64; }
  else if (d % 32 == 0 && d / 32 <= 2) { vec = 1; nch = d / 32; }
}
#define LN_SHAPES(X) X(8, 1) X(8, 2) X(8, 3) X(8, 4) X(4, 1) X(4, 3) X(2, 1) X(2, 3) X(1, 1) X(1, 2)

// ------------------------------------------------------------------ LayerNorm
constexpr int LN_MAXQ_ALL = 32;  // d <= 1024

template <int LN_MAXQ>
__global__ void ln_fwd_k(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                         int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    float v[LN_MAXQ];
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      v[q] = 0.f;
      if (c < d) {
        float x = U[r * d + c];
        if (addx) x += ld_as_f32(addx, r * d + c, dt);
        v[q] = x;
        s += x;
      }
    }
    const float mean = warp_sum(s) / d;
    float s2 = 0.f;
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      if (c < d) { float t = v[q] - mean; s2 += t * t; }
    }
    const float rs = rsqrtf(warp_sum(s2) / d + eps);
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      if (c < d) {
        float y = (v[q] - mean) * rs * ld_as_f32(gamma, c, pdt) + ld_as_f32(beta, c, pdt);
        st_from_f32(Y, r * d + c, dt, y);
        if (Rsave) st_from_f32(Rsave, r * d + c, dt, v[q]);
      }
    }
    if (lane == 0) { mu[r] = mean; rstd[r] = rs; }
  }
}
static cudaError_t ln_fwd_generic(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                   int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt, cudaStream_t st) {
  if (d > 32 * LN_MAXQ_ALL) return cudaErrorInvalidValue;
  const int nb = nblocks(rows, 8, 148 * 64);
  if (d <= 128) pdl_launch(ln_fwd_k<4>, nb, 256, 0, st, U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  else if (d <= 256) pdl_launch(ln_fwd_k<8>, nb, 256, 0, st, U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  else pdl_launch(ln_fwd_k<32>, nb, 256, 0, st, U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  ++g_launches;
  return cudaGetLastError();
}

template <int LN_MAXQ>
__global__ void ln_bwd_k(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                         const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                         float* part, int64_t rows_per_block) {
  pdl_entry();
  __shared__ float sg[8][2][256];   // per-warp partials for one 256-column slab
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  const int64_t r0 = blockIdx.x * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  float pg[LN_MAXQ], pb[LN_MAXQ];
#pragma unroll
  for (int q = 0; q < LN_MAXQ; ++q) { pg[q] = 0.f; pb[q] = 0.f; }
  for (int64_t r = r0 + w; r < r1; r += 8) {
    float xh[LN_MAXQ], gy[LN_MAXQ];
    float s1 = 0.f, s2 = 0.f;
    const float m_ = mu[r], rs = rstd[r];
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      xh[q] = 0.f; gy[q] = 0.f;
      if (c < d) {
        float dy = ld_as_f32(dY, r * d + c, dydt);
        xh[q] = (ld_as_f32(Rsave, r * d + c, dt) - m_) * rs;
        gy[q] = dy * ld_as_f32(gamma, c, pdt);
        pg[q] += dy * xh[q];
        pb[q] += dy;
        s1 += gy[q];
        s2 += gy[q] * xh[q];
      }
    }
    s1 = warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      if (c < d) {
        float v = rs * (gy[q] - s1 - xh[q] * s2);
        st_from_f32(dR, r * d + c, dt, v);
        if (acc_mode) {
          float vr = ld_as_f32(dR, r * d + c, dt);   // the stored (rounded) value feeds the residual path
          if (acc_mode == 1) acc[r * d + c] = vr; else acc[r * d + c] += vr;
        }
      }
    }
  }
  // block reduction of the dgamma / dbeta partials in fixed warp order
  for (int slab = 0; slab < d; slab += 256) {
#pragma unroll
    for (int q = 0; q < LN_MAXQ; ++q) {
      int c = lane + 32 * q;
      if (c >= slab && c < slab + 256 && c < d) { sg[w][0][c - slab] = pg[q]; sg[w][1][c - slab] = pb[q]; }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 256 && slab + c < d; c += blockDim.x) {
      float a = 0.f, b = 0.f;
      for (int ww = 0; ww < 8; ++ww) { a += sg[ww][0][c]; b += sg[ww][1][c]; }
      part[(int64_t)blockIdx.x * 2 * d + slab + c] = a;
      part[(int64_t)blockIdx.x * 2 * d + d + slab + c] = b;
    }
    __syncthreads();
  }
}

// Deterministic column sums of a partials matrix part[nparts][n]: block (32 cols x 32 part-strides); thread
// (x, y) sums parts y, y + 32, ... in order, then warp 0 adds the 32 strides in order.  Fixed order at any grid.
__global__ void __launch_bounds__(1024) part_sum_k(const float* __restrict__ part, int nparts, int n,
                                                   float* __restrict__ out0, int n0, float* __restrict__ out1,
                                                   int n1, float* __restrict__ out2, float out2_scale) {
  pdl_entry();
  __shared__ float sm[32][33];
  const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + x;
  float s = 0.f;
  if (c < n) {
    int p = y;
    for (; p + 96 < nparts; p += 128) {   // 4 independent loads in flight, summed in index order
      const float a = part[(int64_t)p * n + c], b = part[(int64_t)(p + 32) * n + c];
      const float d = part[(int64_t)(p + 64) * n + c], e = part[(int64_t)(p + 96) * n + c];
      s = (((s + a) + b) + d) + e;
    }
    for (; p < nparts; p += 32) s += part[(int64_t)p * n + c];
  }
  sm[y][x] = s;
  __syncthreads();
  if (y == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) t += sm[k][x];
    // columns [0, n0) -> out0 +=, [n0, n0 + n1) -> out1 +=, column n0 + n1 -> *out2 = scale * sum
    if (c < n0) { if (out0) out0[c] += t; }
    else if (c < n0 + n1) { if (out1) out1[c - n0] += t; }
    else if (c == n0 + n1 && out2) *out2 = t * out2_scale;
  }
}
static void part_sum(const float* part, int nparts, int n, float* out0, int n0, float* out1, int n1, float* out2,
                     float out2_scale, cudaStream_t st) {
  pdl_launch(part_sum_k, (n + 31) / 32, 1024, 0, st, part, nparts, n, out0, n0, out1, n1, out2, out2_scale);
  ++g_launches;
}
cudaError_t rows_sum_add(const float* part, int nparts, int n, float* out, cudaStream_t st) {
  part_sum(part, nparts, n, out, n, nullptr, 0, nullptr, 0.f, st);
  return cudaGetLastError();
}

static cudaError_t ln_bwd_generic(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                   const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                   float* dgamma, float* dbeta, float* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (d > 32 * LN_MAXQ_ALL) return cudaErrorInvalidValue;
  int nb = (int)std::min<int64_t>((rows + 63) / 64, 148 * 4);
  nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * 2 * d)));
  if (nb < 1) return cudaErrorInvalidValue;
  int64_t rpb = (rows + nb - 1) / nb;
  nb = (int)((rows + rpb - 1) / rpb);
  if (d <= 128)
    pdl_launch(ln_bwd_k<4>, nb, 256, 0, st, dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  else if (d <= 256)
    pdl_launch(ln_bwd_k<8>, nb, 256, 0, st, dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  else
    pdl_launch(ln_bwd_k<32>, nb, 256, 0, st, dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  ++g_launches;
  part_sum(scratch, nb, 2 * d, dgamma, d, dbeta, d, nullptr, 0.f, st);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ LayerNorm, several rows per warp (bf16, d = 8 LPR)
// A row is LPR lanes x 8 columns (16-B bf16 / 32-B fp32 accesses); a warp holds 32 / LPR rows per pass and
// UR passes per iteration, so UR * 32 / LPR rows of loads are in flight per warp.  Row reductions are
// shuffles inside the LPR-lane segment (fixed order: deterministic).
template <int LPR>
__device__ __forceinline__ float seg_sum(float v) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void ld8f(const float* p, float* o) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p)), b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void ld8b(const __nv_bfloat16* p, float* o) { VIO<8, __nv_bfloat16>::ld(p, o); }
template <typename TD> __device__ __forceinline__ void ld8(const TD* p, float* o);
template <> __device__ __forceinline__ void ld8<float>(const float* p, float* o) { ld8f(p, o); }
template <> __device__ __forceinline__ void ld8<__nv_bfloat16>(const __nv_bfloat16* p, float* o) { ld8b(p, o); }

template <int LPR, int UR>
__global__ void __launch_bounds__(256) ln_fwd_r(const float* __restrict__ U, const __nv_bfloat16* __restrict__ addx,
                                                const __nv_bfloat16* __restrict__ gamma,
                                                const __nv_bfloat16* __restrict__ beta, float eps, int64_t rows,
                                                __nv_bfloat16* __restrict__ Y, __nv_bfloat16* __restrict__ Rsave,
                                                float* __restrict__ mu, float* __restrict__ rstd) {
  pdl_entry();
  constexpr int d = 8 * LPR, RPW = 32 / LPR, RPI = RPW * UR;
  const int lane = threadIdx.x & 31, sub = lane / LPR, c = (lane % LPR) * 8;
  float g[8], b[8];
  ld8b(gamma + c, g);
  ld8b(beta + c, b);
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + threadIdx.x / 32) * RPI; r0 < rows; r0 += nw * RPI) {
    float v[UR][8];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t r = r0 + u * RPW + sub;
      if (r < rows) {
        ld8f(U + r * d + c, v[u]);
        if (addx) {
          float x[8];
          ld8b(addx + r * d + c, x);
#pragma unroll
          for (int t = 0; t < 8; ++t) v[u][t] += x[t];
        }
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) v[u][t] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t r = r0 + u * RPW + sub;
      float s = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) s += v[u][t];
      const float mean = seg_sum<LPR>(s) / d;
      float s2 = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) { const float q = v[u][t] - mean; s2 += q * q; }
      const float rs = rsqrtf(seg_sum<LPR>(s2) / d + eps);
      if (r < rows) {
        float y[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) y[t] = (v[u][t] - mean) * rs * g[t] + b[t];
        VIO<8, __nv_bfloat16>::st(Y + r * d + c, y);
        if (Rsave) VIO<8, __nv_bfloat16>::st(Rsave + r * d + c, v[u]);
        if (c == 0) { mu[r] = mean; rstd[r] = rs; }
      }
    }
  }
}

#ifndef LNB_NB
#define LNB_NB 4   // operand buffers of the LayerNorm backward: 3 iterations of loads in flight ahead of the one
                   // computed (same box: C5 +2.6 %, C4 +0.7 % over 1 ahead; 128 registers keep 2 blocks an SM)
#endif
template <int LPR, int UR, typename TD>
__global__ void __launch_bounds__(256) ln_bwd_r(const TD* __restrict__ dY, const __nv_bfloat16* __restrict__ Rsave,
                                                const float* __restrict__ mu, const float* __restrict__ rstd,
                                                const __nv_bfloat16* __restrict__ gamma, int64_t rows,
                                                __nv_bfloat16* __restrict__ dR, float* __restrict__ acc, int acc_mode,
                                                float* __restrict__ part, int64_t rows_per_block,
                                                const float* __restrict__ vdz = nullptr,
                                                const __nv_bfloat16* __restrict__ vw = nullptr, int vm = 1) {
  pdl_entry();
  constexpr int d = 8 * LPR, RPW = 32 / LPR, RPI = RPW * UR;
  __shared__ float sred[8][2][d];
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32, sub = lane / LPR, c = (lane % LPR) * 8;
  const int64_t rb0 = blockIdx.x * rows_per_block, rb1 = min(rows, rb0 + rows_per_block);
  float g[8], pg[8], pb[8], wv[8];
  ld8b(gamma + c, g);
  // vdz: the head's upstream gradient is never stored -- row r of dY is bf16(dz_b / m * w) with b = r / m
  // (F13 / B1, the same arithmetic as head_v), formed here from the per-sample dz and the head weight
  if (vdz) ld8b(vw + c, wv);
#pragma unroll
  for (int t = 0; t < 8; ++t) { pg[t] = 0.f; pb[t] = 0.f; }
  // raw operands of one iteration (bf16 dY and R as 16-B words): the next iteration's are loaded while this
  // one is computed (software pipelining: two iterations of loads in flight per warp)
  constexpr bool RAWP = true;   // bf16 dY: one 16-B word; fp32 dY: two (ry, ry2)
  constexpr bool F32DY = std::is_same<TD, float>::value;
  constexpr int NB = LNB_NB;   // iterations of loads in flight (ring of operand buffers)
  uint4 ry[NB][UR], rx[NB][UR], ry2[NB][F32DY ? UR : 1];
  float rm[NB][UR], rq[NB][UR];
  auto fetch = [&](int64_t r0_, int bsl) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t r = r0_ + u * RPW + sub;
      if (r < rb1) {
        if constexpr (F32DY) {
          ry[bsl][u] = __ldcs(reinterpret_cast<const uint4*>(dY + r * d + c));
          ry2[bsl][u] = __ldcs(reinterpret_cast<const uint4*>(dY + r * d + c) + 1);
        } else {
          if (vdz) {
            const float gv = vdz[r / vm] / vm;
            uint32_t o[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(gv * wv[2 * t], gv * wv[2 * t + 1]);
              o[t] = *reinterpret_cast<uint32_t*>(&h2);
            }
            ry[bsl][u] = make_uint4(o[0], o[1], o[2], o[3]);
          } else {
            ry[bsl][u] = __ldg(reinterpret_cast<const uint4*>(dY + r * d + c));
          }
        }
        rx[bsl][u] = __ldg(reinterpret_cast<const uint4*>(Rsave + r * d + c));
        rm[bsl][u] = mu[r];
        rq[bsl][u] = rstd[r];
      } else {
        ry[bsl][u] = make_uint4(0u, 0u, 0u, 0u); rx[bsl][u] = make_uint4(0u, 0u, 0u, 0u);
        if constexpr (F32DY) ry2[bsl][u] = make_uint4(0u, 0u, 0u, 0u);
        rm[bsl][u] = 0.f; rq[bsl][u] = 0.f;
      }
    }
  };
  auto body = [&](int64_t r0, auto BSC) {
    constexpr int BS = decltype(BSC)::value;
    if (r0 + (NB - 1) * 8 * RPI < rb1) fetch(r0 + (NB - 1) * 8 * RPI, (BS + NB - 1) % NB);   // later iterations' operands in flight
    float dy[UR][8], x[UR][8], mr[UR], rr[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t r = r0 + u * RPW + sub;
      if constexpr (F32DY) {
        const uint4 a = ry[BS][u], b = ry2[BS][u];
        dy[u][0] = __uint_as_float(a.x); dy[u][1] = __uint_as_float(a.y); dy[u][2] = __uint_as_float(a.z);
        dy[u][3] = __uint_as_float(a.w); dy[u][4] = __uint_as_float(b.x); dy[u][5] = __uint_as_float(b.y);
        dy[u][6] = __uint_as_float(b.z); dy[u][7] = __uint_as_float(b.w);
      } else if constexpr (RAWP) {
        VIO<8, __nv_bfloat16>::ld(reinterpret_cast<const __nv_bfloat16*>(&ry[BS][u]), dy[u]);
      } else {
        if (r < rb1) ld8<TD>(dY + r * d + c, dy[u]);
        else {
#pragma unroll
          for (int t = 0; t < 8; ++t) dy[u][t] = 0.f;
        }
      }
      VIO<8, __nv_bfloat16>::ld(reinterpret_cast<const __nv_bfloat16*>(&rx[BS][u]), x[u]);
      mr[u] = rm[BS][u];
      rr[u] = rq[BS][u];
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int64_t r = r0 + u * RPW + sub;
      const bool ok = r < rb1;
      const float m_ = mr[u], rs = rr[u];
      float xh[8], gy[8], s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        xh[t] = (x[u][t] - m_) * rs;
        gy[t] = dy[u][t] * g[t];
        pg[t] += dy[u][t] * xh[t];
        pb[t] += dy[u][t];
        s1 += gy[t];
        s2 += gy[t] * xh[t];
      }
      s1 = seg_sum<LPR>(s1) / d;
      s2 = seg_sum<LPR>(s2) / d;
      if (ok) {
        float o[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) o[t] = rs * (gy[t] - s1 - xh[t] * s2);
        uint4 q;
        {
          __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]),
                         h2 = __floats2bfloat162_rn(o[4], o[5]), h3 = __floats2bfloat162_rn(o[6], o[7]);
          q = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                         *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
        }
        *reinterpret_cast<uint4*>(dR + r * d + c) = q;
        if (acc_mode) {   // the stored (rounded) value feeds the residual path
          const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
          float qf[8];
#pragma unroll
          for (int t = 0; t < 4; ++t) { qf[2 * t] = __uint_as_float(qw[t] << 16); qf[2 * t + 1] = __uint_as_float(qw[t] & 0xffff0000u); }
          float* ap = acc + r * d + c;
          if (acc_mode == 1) {
            reinterpret_cast<float4*>(ap)[0] = make_float4(qf[0], qf[1], qf[2], qf[3]);
            reinterpret_cast<float4*>(ap)[1] = make_float4(qf[4], qf[5], qf[6], qf[7]);
          } else {   // acc += dR in L2 (one adder per element)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ap), "f"(qf[0]), "f"(qf[1]), "f"(qf[2]), "f"(qf[3]) : "memory");
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ap + 4), "f"(qf[4]), "f"(qf[5]), "f"(qf[6]), "f"(qf[7]) : "memory");
          }
        }
      }
    }
    };
  const int64_t rs0 = rb0 + (int64_t)w * RPI;
#pragma unroll
  for (int k = 0; k < NB - 1; ++k)
    if (rs0 + k * 8 * RPI < rb1) fetch(rs0 + k * 8 * RPI, k);
  for (int64_t r0 = rs0; r0 < rb1; r0 += NB * 8 * RPI) {   // NB iterations per trip: buffer indices compile-time
    body(r0, std::integral_constant<int, 0>{});
    if (r0 + 8 * RPI < rb1) body(r0 + 8 * RPI, std::integral_constant<int, 1>{});
    if constexpr (NB > 2) { if (r0 + 16 * RPI < rb1) body(r0 + 16 * RPI, std::integral_constant<int, 2 % NB>{}); }
    if constexpr (NB > 3) { if (r0 + 24 * RPI < rb1) body(r0 + 24 * RPI, std::integral_constant<int, 3 % NB>{}); }
  }
  // dgamma / dbeta: lanes with equal columns (xor offsets >= LPR), then the 8 warps in order
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      pg[t] += __shfl_xor_sync(0xffffffffu, pg[t], o);
      pb[t] += __shfl_xor_sync(0xffffffffu, pb[t], o);
    }
  if (sub == 0) {
#pragma unroll
    for (int t = 0; t < 8; ++t) { sred[w][0][c + t] = pg[t]; sred[w][1][c + t] = pb[t]; }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 2 * d; j += blockDim.x) {
    const int which = j / d, cc = j - which * d;
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) s += sred[ww][which][cc];
    part[(int64_t)blockIdx.x * 2 * d + j] = s;
  }
}

// one resident wave: SMs x blocks per SM at the kernel's register / smem occupancy
template <typename K>
static int resident_blocks(K kern, int threads, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1) {
    (void)cudaGetLastError();
    per = 1;
  }
  return sms * per;
}
#ifndef LNB_UR
#define LNB_UR 1   // rows per lane segment per iteration of the LayerNorm backward (loads in flight); 1 measured
                   // best on the same box: C5 +3.8 %, C2 +1.3 %, C3 +1 %, C4 +0.9 % over 2 (fewer registers)
#endif
static int ln_bwd_grid(int lpr, int dydt) {
  static int cache[2][6] = {{0}};
  const int li = lpr == 4 ? 0 : lpr == 8 ? 1 : lpr == 16 ? 2 : 3, ti = dydt == BF16 ? 0 : 1;
  int& v = cache[ti][li];
  if (!v) {
#define LG(L, I) if (li == I) v = ti == 0 ? resident_blocks(ln_bwd_r<L, LNB_UR, __nv_bfloat16>, 256, 0) : resident_blocks(ln_bwd_r<L, LNB_UR, float>, 256, 0);
    LG(4, 0) LG(8, 1) LG(16, 2) LG(32, 3)
#undef LG
  }
  return v;
}
static int ln_lpr(int d) { return (d % 8 == 0 && (d / 8) <= 32 && ((d / 8) & (d / 8 - 1)) == 0) ? d / 8 : 0; }

cudaError_t ln_fwd(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                   int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt, cudaStream_t st) {
  const int lpr = ln_lpr(d);
  if (dt == BF16 && pdt == BF16 && lpr >= 4) {
    const int rpi = (32 / lpr) * 2;   // rows per warp iteration (UR = 2)
    const int nb = nblocks((rows + rpi - 1) / rpi, 8, 148 * 8);
#define LNR(L)                                                                                                    \
    if (lpr == L) pdl_launch(ln_fwd_r<L, 2>, nb, 256, 0, st, U, (const __nv_bfloat16*)addx, (const __nv_bfloat16*)gamma, \
        (const __nv_bfloat16*)beta, eps, rows, (__nv_bfloat16*)Y, (__nv_bfloat16*)Rsave, mu, rstd);
    LNR(4) LNR(8) LNR(16) LNR(32)
#undef LNR
    ++g_launches;
    return cudaGetLastError();
  }
  int vec, nch;
  ln_shape(d, vec, nch);
  if (!vec || pdt != dt) return ln_fwd_generic(U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt, st);
  const int nb = nblocks(rows, 8, 148 * 64);
#define LNF(V, N)                                                                                               \
  if (vec == V && nch == N) {                                                                                   \
    if (dt == BF16)                                                                                             \
      pdl_launch(ln_fwd_v<__nv_bfloat16, V, N>, nb, 256, 0, st, U, (const __nv_bfloat16*)addx, (const __nv_bfloat16*)gamma, \
          (const __nv_bfloat16*)beta, eps, rows, d, (__nv_bfloat16*)Y, (__nv_bfloat16*)Rsave, mu, rstd);       \
    else                                                                                                        \
      pdl_launch(ln_fwd_v<float, V, N>, nb, 256, 0, st, U, (const float*)addx, (const float*)gamma, (const float*)beta, eps, \
          rows, d, (float*)Y, (float*)Rsave, mu, rstd);                                                        \
  }
  LN_SHAPES(LNF)
#undef LNF
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t ln_bwd(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                   const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                   float* dgamma, float* dbeta, float* scratch, size_t scratch_bytes, cudaStream_t st,
                   cudaStream_t st_red, cudaEvent_t ev_red, const float* vdz, const void* vw, int vm) {
  const int lpr = ln_lpr(d);
  if (vdz && !(dt == BF16 && pdt == BF16 && lpr >= 4 && dydt == BF16 && vw && vm > 0)) return cudaErrorNotSupported;
  if (dt == BF16 && pdt == BF16 && lpr >= 4) {
    const int rpi = (32 / lpr) * LNB_UR;
    int nb = (int)std::min<int64_t>((rows + 8 * rpi - 1) / (8 * rpi), ln_bwd_grid(lpr, dydt));
    nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * 2 * d)));
    if (nb >= 1) {
      int64_t rpb = (rows + nb - 1) / nb;
      nb = (int)((rows + rpb - 1) / rpb);
#define LNB2(L)                                                                                                        \
      if (lpr == L) {                                                                                                  \
        if (dydt == BF16)                                                                                              \
          pdl_launch(ln_bwd_r<L, LNB_UR, __nv_bfloat16>, nb, 256, 0, st, (const __nv_bfloat16*)dY, (const __nv_bfloat16*)Rsave, mu, \
              rstd, (const __nv_bfloat16*)gamma, rows, (__nv_bfloat16*)dR, acc, acc_mode, scratch, rpb, vdz,        \
              (const __nv_bfloat16*)vw, vm);                                                                   \
        else                                                                                                           \
          pdl_launch(ln_bwd_r<L, LNB_UR, float>, nb, 256, 0, st, (const float*)dY, (const __nv_bfloat16*)Rsave, mu, rstd,           \
              (const __nv_bfloat16*)gamma, rows, (__nv_bfloat16*)dR, acc, acc_mode, scratch, rpb,                   \
              (const float*)nullptr, (const __nv_bfloat16*)nullptr, 1);                                         \
      }
      LNB2(4) LNB2(8) LNB2(16) LNB2(32)
#undef LNB2
      ++g_launches;
      cudaStream_t sr = st;
      if (st_red && ev_red && st_red != st) {   // dR is what st needs next; the parameter sums can trail
        cudaEventRecord(ev_red, st);
        cudaStreamWaitEvent(st_red, ev_red, 0);
        sr = st_red;
      }
      part_sum(scratch, nb, 2 * d, dgamma, d, dbeta, d, nullptr, 0.f, sr);
      return cudaGetLastError();
    }
  }
  int vec, nch;
  ln_shape(d, vec, nch);
  if (!vec || pdt != dt)
    return ln_bwd_generic(dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, dgamma, dbeta,
                          scratch, scratch_bytes, st);
  int nb = (int)std::min<int64_t>((rows + 63) / 64, 148 * 4);
  nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * 2 * d)));
  if (nb < 1) return cudaErrorInvalidValue;
  int64_t rpb = (rows + nb - 1) / nb;
  nb = (int)((rows + rpb - 1) / rpb);
  const size_t sm = (size_t)16 * d * sizeof(float);
  if (sm > 48 * 1024)
    return ln_bwd_generic(dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, dgamma, dbeta,
                          scratch, scratch_bytes, st);
#define LNB(V, N)                                                                                                   \
  if (vec == V && nch == N) {                                                                                       \
    if (dt == BF16) {                                                                                               \
      if (dydt == BF16)                                                                                             \
        pdl_launch(ln_bwd_v<__nv_bfloat16, __nv_bfloat16, V, N>, nb, 256, sm, st, (const __nv_bfloat16*)dY,                 \
            (const __nv_bfloat16*)Rsave, mu, rstd, (const __nv_bfloat16*)gamma, rows, d, (__nv_bfloat16*)dR, acc,   \
            acc_mode, scratch, rpb);                                                                                \
      else                                                                                                          \
        pdl_launch(ln_bwd_v<float, __nv_bfloat16, V, N>, nb, 256, sm, st, (const float*)dY, (const __nv_bfloat16*)Rsave,    \
            mu, rstd, (const __nv_bfloat16*)gamma, rows, d, (__nv_bfloat16*)dR, acc, acc_mode, scratch, rpb);       \
    } else {                                                                                                        \
      pdl_launch(ln_bwd_v<float, float, V, N>, nb, 256, sm, st, (const float*)dY, (const float*)Rsave, mu, rstd,            \
          (const float*)gamma, rows, d, (float*)dR, acc, acc_mode, scratch, rpb);                                   \
    }                                                                                                               \
  }
  LN_SHAPES(LNB)
#undef LNB
  ++g_launches;
  part_sum(scratch, nb, 2 * d, dgamma, d, dbeta, d, nullptr, 0.f, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ column sums
__global__ void colsum_part_k(const void* src, int dt, int64_t rows, int cols, int64_t ld, int64_t rpc, float* part) {
  pdl_entry();
  __shared__ float sm[8][33];
  const int cx = threadIdx.x % 32, ry = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + cx;
  const int64_t r0 = blockIdx.y * rpc, r1 = min(rows, r0 + rpc);
  float s = 0.f;
  if (c < cols)
    for (int64_t r = r0 + ry; r < r1; r += 8) s += ld_as_f32(src, r * ld + c, dt);
  sm[ry][cx] = s;
  __syncthreads();
  if (ry == 0 && c < cols) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += sm[k][cx];
    part[(int64_t)blockIdx.y * cols + c] = t;
  }
}
// vectorised: thread (tx, ty) owns 8 consecutive columns tx*8.. of a 256-column slab and rows ty, ty+8, ...
template <typename T>
__global__ void __launch_bounds__(256) colsum8_part_k(const T* __restrict__ src, int64_t rows, int cols, int64_t ld,
                                                      int64_t rpc, float* __restrict__ part) {
  pdl_entry();
  __shared__ float sm[8][257];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int c = blockIdx.x * 256 + tx * 8;
  const int64_t r0 = blockIdx.y * rpc, r1 = min(rows, r0 + rpc);
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < cols) {
    int64_t r = r0 + ty;
    for (; r + 24 < r1; r += 32) {     // 4 independent loads in flight
      float v0[8], v1[8], v2[8], v3[8];
      VIO<8, T>::ld(src + r * ld + c, v0);
      VIO<8, T>::ld(src + (r + 8) * ld + c, v1);
      VIO<8, T>::ld(src + (r + 16) * ld + c, v2);
      VIO<8, T>::ld(src + (r + 24) * ld + c, v3);
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] += (v0[t] + v1[t]) + (v2[t] + v3[t]);
    }
    for (; r < r1; r += 8) {
      float v0[8];
      VIO<8, T>::ld(src + r * ld + c, v0);
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] += v0[t];
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) sm[ty][tx * 8 + t] = a[t];
  __syncthreads();
  const int cc = blockIdx.x * 256 + threadIdx.x;
  if (cc < cols) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += sm[k][threadIdx.x];
    part[(int64_t)blockIdx.y * cols + cc] = t;
  }
}

// cols <= 2048, cols % 8 == 0: one block covers every column: CT = cols / 8 column-threads (8 columns each, 16-B
// loads) x RT = 256 / CT row-threads; the RT partial rows are added in fixed order through shared memory.
__global__ void __launch_bounds__(256) colsum_all_k(const __nv_bfloat16* __restrict__ src, int64_t rows, int cols,
                                                    int64_t ld, int64_t rpc, float* __restrict__ part) {
  pdl_entry();
  extern __shared__ float csm[];   // [RT][cols]
  const int CT = cols / 8, RT = 256 / CT;
  const int ct = threadIdx.x % CT, ry = threadIdx.x / CT, c = ct * 8;
  const int64_t r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
  if (ry < RT) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int64_t r = r0 + ry;
    for (; r + 3 * RT < r1; r += 4 * RT) {   // 4 independent 16-B loads in flight
      float v0[8], v1[8], v2[8], v3[8];
      VIO<8, __nv_bfloat16>::ld(src + r * ld + c, v0);
      VIO<8, __nv_bfloat16>::ld(src + (r + RT) * ld + c, v1);
      VIO<8, __nv_bfloat16>::ld(src + (r + 2 * RT) * ld + c, v2);
      VIO<8, __nv_bfloat16>::ld(src + (r + 3 * RT) * ld + c, v3);
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] += (v0[t] + v1[t]) + (v2[t] + v3[t]);
    }
    for (; r < r1; r += RT) {
      float v0[8];
      VIO<8, __nv_bfloat16>::ld(src + r * ld + c, v0);
#pragma unroll
      for (int t = 0; t < 8; ++t) a[t] += v0[t];
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) csm[ry * cols + c + t] = a[t];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < cols; j += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < RT; ++k) s += csm[k * cols + j];
    part[(int64_t)blockIdx.x * cols + j] = s;
  }
}

cudaError_t colsum_add(const void* src, int dt, int64_t rows, int cols, int64_t ld, float* out, float* scratch,
                       size_t scratch_bytes, cudaStream_t st) {
  const int es = dt == F32 ? 4 : 2;
  if (dt == BF16 && cols % 8 == 0 && cols <= 2048 && ld % 8 == 0 && ((uintptr_t)src % 16) == 0) {
    const int CT = cols / 8, RT = 256 / CT;
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(rows / (4 * RT), 4 * 148));
    nch = std::min<int64_t>(nch, (int64_t)(scratch_bytes / (sizeof(float) * cols)));
    if (nch >= 1) {
      int64_t rpc = (rows + nch - 1) / nch;
      nch = (rows + rpc - 1) / rpc;
      if (nch < 1) nch = 1;
      pdl_launch(colsum_all_k, (unsigned)nch, 256, (size_t)RT * cols * sizeof(float), st, (const __nv_bfloat16*)src, rows, cols,
                                                                                   ld, rpc, scratch);
      ++g_launches;
      part_sum(scratch, (int)nch, cols, out, cols, nullptr, 0, nullptr, 0.f, st);
      return cudaGetLastError();
    }
  }
  if (cols % 8 == 0 && ld % 8 == 0 && ((uintptr_t)src % (8 * es)) == 0) {
    const int cb = (cols + 255) / 256;
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(rows / 64, std::max(1, 4 * 148 / cb)));
    nch = std::min<int64_t>(nch, (int64_t)(scratch_bytes / (sizeof(float) * cols)));
    if (nch >= 1) {
      int64_t rpc = (rows + nch - 1) / nch;
      nch = (rows + rpc - 1) / rpc;
      if (nch < 1) nch = 1;
      if (dt == F32)
        pdl_launch(colsum8_part_k<float>, dim3(cb, (unsigned)nch), 256, 0, st, (const float*)src, rows, cols, ld, rpc, scratch);
      else
        pdl_launch(colsum8_part_k<__nv_bfloat16>, dim3(cb, (unsigned)nch), 256, 0, st, (const __nv_bfloat16*)src, rows, cols,
                                                                                ld, rpc, scratch);
      ++g_launches;
      part_sum(scratch, (int)nch, cols, out, cols, nullptr, 0, nullptr, 0.f, st);
      return cudaGetLastError();
    }
  }
  int cb = (cols + 31) / 32;
  int64_t nch = std::max<int64_t>(1, std::min<int64_t>(rows / 256, std::max(1, 296 / cb)));
  nch = std::min<int64_t>(nch, (int64_t)(scratch_bytes / (sizeof(float) * cols)));
  if (nch < 1) return cudaErrorInvalidValue;
  int64_t rpc = (rows + nch - 1) / nch;
  nch = (rows + rpc - 1) / rpc;
  if (nch < 1) nch = 1;
  pdl_launch(colsum_part_k, dim3(cb, (unsigned)nch), 256, 0, st, src, dt, rows, cols, ld, rpc, scratch);
  ++g_launches;
  part_sum(scratch, (int)nch, cols, out, cols, nullptr, 0, nullptr, 0.f, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ softmax
__global__ void softmax_rows_k(const float* S, void* P, int dt, int64_t rows, int n, int ld) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* s = S + r * ld;
    float mx = -INFINITY;
    for (int c = lane; c < n; c += 32) mx = fmaxf(mx, s[c]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int c = lane; c < n; c += 32) sum += __expf(s[c] - mx);
    const float inv = 1.f / warp_sum(sum);
    for (int c = lane; c < n; c += 32) st_from_f32(P, r * ld + c, dt, __expf(s[c] - mx) * inv);
  }
}
cudaError_t softmax_rows(const float* S, void* P, int dt, int64_t rows, int n, int ld, cudaStream_t st) {
  pdl_launch(softmax_rows_k, nblocks(rows, 8, 148 * 64), 256, 0, st, S, P, dt, rows, n, ld);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void softmax_bwd_k(const void* P, const float* dP, void* dS, int dt, int64_t rows, int n, int ld,
                              float scale) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    float s = 0.f;
    for (int c = lane; c < n; c += 32) s += ld_as_f32(P, r * ld + c, dt) * dP[r * ld + c];
    s = warp_sum(s);
    for (int c = lane; c < n; c += 32) {
      float p = ld_as_f32(P, r * ld + c, dt);
      st_from_f32(dS, r * ld + c, dt, scale * p * (dP[r * ld + c] - s));
    }
  }
}
cudaError_t softmax_bwd(const void* P, const float* dP, void* dS, int dt, int64_t rows, int n, int ld, float scale,
                        cudaStream_t st) {
  pdl_launch(softmax_bwd_k, nblocks(rows, 8, 148 * 64), 256, 0, st, P, dP, dS, dt, rows, n, ld, scale);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ DCN backward elementwise
__global__ void dcn_bwd_elem_k(const void* dT, const void* X, const void* A, void* dA, float* acc, int dt, int64_t n) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    float g = ld_as_f32(dT, t, dt), x = ld_as_f32(X, t, dt), a = ld_as_f32(A, t, dt);
    st_from_f32(dA, t, dt, g * x);
    acc[t] += g * a + g;
  }
}
cudaError_t dcn_bwd_elem(const void* dT, const void* X, const void* A, void* dA, float* acc, int dt, int64_t n,
                         cudaStream_t st) {
  pdl_launch(dcn_bwd_elem_k, nblocks(n), 256, 0, st, dT, X, A, dA, acc, dt, n);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ conv, banded shared-memory stencils
// Block = one sample b and a band of RB = 8 output rows; the band + halo rows of the input live in smem
// (zero padded), each thread computes 8 consecutive outputs of one row.  d % 8 == 0, d <= 1024.
constexpr int CV_RB = 8;
template <typename T, int K, bool FLIP>
__global__ void __launch_bounds__(256) conv_band_k(const T* __restrict__ in, const T* __restrict__ Kp, int C, int m,
                                                   int d, T* __restrict__ outT, float* __restrict__ outAcc, int nbatch) {
  pdl_entry();
  constexpr int R = (K - 1) / 2;
  extern __shared__ float band[];          // [(RB + 2R) rows][d + 2R]
  __shared__ float kb[K * K];
  const int W = d + 2 * R;
  for (int t = threadIdx.x; t < K * K; t += blockDim.x) {
    float sacc = 0.f;
    for (int c = 0; c < C; ++c) sacc += tof<T>(Kp[c * K * K + t]);
    kb[t] = sacc / C;
  }
  const int rows_in = CV_RB + 2 * R;
  const int nbm = (m + CV_RB - 1) / CV_RB;
  for (int64_t band_i = blockIdx.x; band_i < (int64_t)nbm * nbatch; band_i += gridDim.x) {
  const int b = (int)(band_i / nbm), i0 = (int)(band_i % nbm) * CV_RB;
  __syncthreads();
  for (int e = threadIdx.x; e < rows_in * (d / 8); e += blockDim.x) {
    const int rr = e / (d / 8), cc = (e % (d / 8)) * 8;
    const int gi = i0 - R + rr;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (gi >= 0 && gi < m) VIO<8, T>::ld(in + ((int64_t)b * m + gi) * d + cc, v);
#pragma unroll
    for (int t = 0; t < 8; ++t) band[rr * W + R + cc + t] = v[t];
  }
  for (int e = threadIdx.x; e < rows_in * 2 * R; e += blockDim.x) {   // zero the left / right halo columns
    const int rr = e / (2 * R), q = e % (2 * R);
    band[rr * W + (q < R ? q : d + q)] = 0.f;
  }
  __syncthreads();
  // thread <-> output column j (consecutive threads, consecutive smem words: conflict-free); each thread
  // walks down the band's rows (RPT rows per thread when d < blockDim)
  const int cpb = d < (int)blockDim.x ? d : (int)blockDim.x;      // columns per pass
  const int rgroups = (int)blockDim.x / cpb;                       // row groups (d < 256)
  const int rpt = (CV_RB + rgroups - 1) / rgroups;
  const int rg = threadIdx.x / cpb;
  for (int j = threadIdx.x % cpb; j < d; j += cpb) {
    if (rg >= rgroups) break;
    const int r0 = rg * rpt, r1 = min(CV_RB, r0 + rpt);
    for (int ri = r0; ri < r1; ++ri) {
      const int gi = i0 + ri;
      if (gi >= m) break;
      float o = 0.f;
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const float* row = band + (ri + (FLIP ? 2 * R - a : a)) * W + j;
#pragma unroll
        for (int e2 = 0; e2 < K; ++e2) o += kb[a * K + e2] * row[FLIP ? 2 * R - e2 : e2];
      }
      const int64_t off = ((int64_t)b * m + gi) * d + j;
      if (outAcc) outAcc[off] += o;
      else outT[off] = fromf<T>(o);
    }
  }
  }
}

// dK[a][e] partials: block = (band of sample b): sum over its outputs of dT[i][j] * X[i+a-R][j+e-R]
template <typename T, int K>
__global__ void __launch_bounds__(256) conv_wgrad_band_k(const T* __restrict__ dT, const T* __restrict__ X, int m,
                                                         int d, float* __restrict__ part, int nbatch) {
  pdl_entry();
  constexpr int R = (K - 1) / 2;
  extern __shared__ float band[];          // X band [(RB + 2R)][d + 2R]
  __shared__ float red[K * K][8];
  const int W = d + 2 * R, rows_in = CV_RB + 2 * R;
  const int nbm = (m + CV_RB - 1) / CV_RB;
  float acc[K * K];
#pragma unroll
  for (int q = 0; q < K * K; ++q) acc[q] = 0.f;
  for (int64_t band_i = blockIdx.x; band_i < (int64_t)nbm * nbatch; band_i += gridDim.x) {
  const int b = (int)(band_i / nbm), i0 = (int)(band_i % nbm) * CV_RB;
  __syncthreads();
  for (int e = threadIdx.x; e < rows_in * (d / 8); e += blockDim.x) {
    const int rr = e / (d / 8), cc = (e % (d / 8)) * 8;
    const int gi = i0 - R + rr;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (gi >= 0 && gi < m) VIO<8, T>::ld(X + ((int64_t)b * m + gi) * d + cc, v);
#pragma unroll
    for (int t = 0; t < 8; ++t) band[rr * W + R + cc + t] = v[t];
  }
  for (int e = threadIdx.x; e < rows_in * 2 * R; e += blockDim.x) {
    const int rr = e / (2 * R), q = e % (2 * R);
    band[rr * W + (q < R ? q : d + q)] = 0.f;
  }
  __syncthreads();
  const int cpb = d < (int)blockDim.x ? d : (int)blockDim.x;
  const int rgroups = (int)blockDim.x / cpb;
  const int rpt = (CV_RB + rgroups - 1) / rgroups;
  const int rg = threadIdx.x / cpb;
  for (int j = threadIdx.x % cpb; j < d && rg < rgroups; j += cpb) {
    const int r0 = rg * rpt, r1 = min(CV_RB, r0 + rpt);
    for (int ri = r0; ri < r1; ++ri) {
      const int gi = i0 + ri;
      if (gi >= m) break;
      const float g = tof<T>(dT[((int64_t)b * m + gi) * d + j]);
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const float* row = band + (ri + a) * W + j;
#pragma unroll
        for (int e2 = 0; e2 < K; ++e2) acc[a * K + e2] += g * row[e2];
      }
    }
  }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
#pragma unroll
  for (int q = 0; q < K * K; ++q) {
    const float v = warp_sum(acc[q]);
    if (lane == 0) red[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < K * K) {
    float v = 0.f;
    for (int ww = 0; ww < 8; ++ww) v += red[threadIdx.x][ww];
    part[(int64_t)blockIdx.x * K * K + threadIdx.x] = v;
  }
}

// Whole-sample variant: the sample's m x d image (+ zero halo) is staged in shared memory (as T) with all
// 16-B loads in flight; thread <-> column j, a K-row register window slides down the rows.
// MODE 0: T_out = Kbar (*) X;  1: acc += flip(Kbar) (*) dT;  2: dK partials += sum dT[i][j] X[i+a-R][j+e-R].
template <typename T, int K, int MODE>
__global__ void __launch_bounds__(256) conv_sample_k(const T* __restrict__ img, const T* __restrict__ other,
                                                     const T* __restrict__ Kp, int C, int B, int m, int d,
                                                     T* __restrict__ outT, float* __restrict__ outAcc,
                                                     float* __restrict__ part) {
  pdl_entry();
  constexpr int R = (K - 1) / 2;
  extern __shared__ __align__(16) unsigned char conv_smem[];
  T* S = reinterpret_cast<T*>(conv_smem);            // [(m + 2R)][W]
  __shared__ float kb[K * K];
  __shared__ float red[K * K][8];
  const int W = d + 2 * R;
  if (MODE != 2) {
    for (int t = threadIdx.x; t < K * K; t += blockDim.x) {
      float sacc = 0.f;
      for (int c = 0; c < C; ++c) sacc += tof<T>(Kp[c * K * K + t]);
      kb[t] = sacc / C;
    }
  }
  // zero the halo once (rows 0..R-1, m+R..m+2R-1, and columns 0..R-1, d+R..d+2R-1 of every row)
  for (int e = threadIdx.x; e < (m + 2 * R) * W; e += blockDim.x) {
    const int rr = e / W, cc = e % W;
    if (rr < R || rr >= m + R || cc < R || cc >= d + R) S[e] = fromf<T>(0.f);
  }
  float wacc[K * K];
#pragma unroll
  for (int q = 0; q < K * K; ++q) wacc[q] = 0.f;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    __syncthreads();
    // stage the sample (8 elements per 16-B load); interior only
    const T* src = img + (int64_t)b * m * d;
    for (int e = threadIdx.x; e < m * (d / 8); e += blockDim.x) {
      const int rr = e / (d / 8), cc = (e % (d / 8)) * 8;
      float v[8];
      VIO<8, T>::ld(src + (int64_t)rr * d + cc, v);
      T* dst = S + (rr + R) * W + R + cc;
#pragma unroll
      for (int t = 0; t < 8; ++t) dst[t] = fromf<T>(v[t]);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      // window rows: w[a][e] = S[i + a][j + e] (padded coordinates)
      float w[K][K];
#pragma unroll
      for (int a = 0; a < K - 1; ++a)
#pragma unroll
        for (int e = 0; e < K; ++e) w[a + 1][e] = tof<T>(S[a * W + j + e]);
      if (MODE == 1) {
        // dgrad: 8 rows of outputs in registers, then their 8 accumulator loads in flight together
        for (int i0 = 0; i0 < m; i0 += 8) {
          float o8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = i0 + u;
            o8[u] = 0.f;
            if (i < m) {
#pragma unroll
              for (int a = 0; a < K - 1; ++a)
#pragma unroll
                for (int e = 0; e < K; ++e) w[a][e] = w[a + 1][e];
#pragma unroll
              for (int e = 0; e < K; ++e) w[K - 1][e] = tof<T>(S[(i + K - 1) * W + j + e]);
#pragma unroll
              for (int a = 0; a < K; ++a)
#pragma unroll
                for (int e = 0; e < K; ++e) o8[u] += kb[(K - 1 - a) * K + (K - 1 - e)] * w[a][e];
            }
          }
          float c8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            c8[u] = (i0 + u < m) ? __ldcg(outAcc + ((int64_t)b * m + i0 + u) * d + j) : 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i0 + u < m) outAcc[((int64_t)b * m + i0 + u) * d + j] = c8[u] + o8[u];
        }
        continue;
      }
      for (int i = 0; i < m; ++i) {
#pragma unroll
        for (int a = 0; a < K - 1; ++a)
#pragma unroll
          for (int e = 0; e < K; ++e) w[a][e] = w[a + 1][e];
#pragma unroll
        for (int e = 0; e < K; ++e) w[K - 1][e] = tof<T>(S[(i + K - 1) * W + j + e]);
        const int64_t off = ((int64_t)b * m + i) * d + j;
        if (MODE == 0) {
          float o = 0.f;
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int e = 0; e < K; ++e) o += kb[a * K + e] * w[a][e];
          outT[off] = fromf<T>(o);
        } else if (MODE == 1) {
          float o = 0.f;
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int e = 0; e < K; ++e) o += kb[(K - 1 - a) * K + (K - 1 - e)] * w[a][e];
          outAcc[off] += o;
        } else {
          const float g = tof<T>(other[off]);
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int e = 0; e < K; ++e) wacc[a * K + e] += g * w[a][e];
        }
      }
    }
  }
  if (MODE == 2) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x / 32;
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      const float v = warp_sum(wacc[q]);
      if (lane == 0) red[q][wi] = v;
    }
    __syncthreads();
    if (threadIdx.x < K * K) {
      float v = 0.f;
      for (int ww = 0; ww < (int)(blockDim.x / 32); ++ww) v += red[threadIdx.x][ww];
      part[(int64_t)blockIdx.x * K * K + threadIdx.x] = v;
    }
  }
}

template <typename T, int K, int MODE>
static cudaError_t conv_sample_launch(const void* img, const void* other, const void* Kp, int C, int B, int m, int d,
                                      void* outT, float* outAcc, float* part, int grid, cudaStream_t st) {
  constexpr int R = (K - 1) / 2;
  const size_t sm = (size_t)(m + 2 * R) * (d + 2 * R) * sizeof(T);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_sample_k<T, K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  pdl_launch(conv_sample_k<T, K, MODE>, grid, 256, sm, st, (const T*)img, (const T*)other, (const T*)Kp, C, B, m, d, (T*)outT,
                                                   outAcc, part);
  ++g_launches;
  return cudaGetLastError();
}
static bool conv_sample_ok(int k, int m, int d, int es) {
  return k == 3 && d % 8 == 0 && (size_t)(m + 2) * (d + 2) * es <= 200 * 1024;
}

template <typename T, int K>
static cudaError_t conv_band_launch(const void* in, const void* Kp, int C, int B, int m, int d, void* outT, float* outAcc,
                                    bool flip, cudaStream_t st) {
  constexpr int R = (K - 1) / 2;
  const size_t sm = (size_t)(CV_RB + 2 * R) * (d + 2 * R) * sizeof(float);
  const int64_t bands = (int64_t)((m + CV_RB - 1) / CV_RB) * B;
  const int grid = (int)std::min<int64_t>(bands, 148 * 8);
  if (flip)
    pdl_launch(conv_band_k<T, K, true>, grid, 256, sm, st, (const T*)in, (const T*)Kp, C, m, d, (T*)outT, outAcc, B);
  else
    pdl_launch(conv_band_k<T, K, false>, grid, 256, sm, st, (const T*)in, (const T*)Kp, C, m, d, (T*)outT, outAcc, B);
  ++g_launches;
  return cudaGetLastError();
}
static bool conv_band_ok(int k, int d, int B) { return (k == 3 || k == 5) && d % 8 == 0 && d <= 1024 && B >= 1; }

// ------------------------------------------------------------------ conv, double-buffered whole-sample stencils
// (bf16, 3x3).  One persistent block per SM; sample b's m x d image arrives with one cp.async.bulk copy into
// rows 1..m of a zero-bordered smem image (rows 0 and m+1 stay zero) while the block computes the previous
// sample from the other buffer.  Thread t owns column j = t % d for the rows of its row group; the window
// slides down the rows in registers (three smem loads per output).  MODE 0: T = K * X (bf16).  MODE 1: dX +=
// K^flip * dT by fp32 reductions in L2 (one adder per element).  MODE 2: dK partials sum dT[i][j] X[i+a][j+e]
// (dT read from global, 8 rows in flight).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
#define mbar_wait1(a, parity) mbar_wait_impl<false>((a), (parity), __FILE__, __LINE__)
template <int MODE>
__global__ void __launch_bounds__(512, 1) conv_db_k(const __nv_bfloat16* __restrict__ img, const __nv_bfloat16* __restrict__ other,
                                                    const __nv_bfloat16* __restrict__ Kp, int C, int B, int m, int d,
                                                    __nv_bfloat16* __restrict__ outT, float* __restrict__ outAcc,
                                                    float* __restrict__ part) {
  pdl_entry();
  // smem image: rows 0..m+1 (0 and m+1 zero), dense rows (pitch d): the sample lands with ONE bulk copy;
  // the two edge column-quads read their out-of-image neighbour as 0.
  extern __shared__ __align__(128) unsigned char cdb_smem[];
  __shared__ __align__(8) uint64_t full[2];
  __shared__ float kb[9];
  __shared__ float red[9][16];
  const int P = d;
  const int S = (m + 2) * P;   // elements per buffer
  __nv_bfloat16* buf0 = reinterpret_cast<__nv_bfloat16*>(cdb_smem);
  if (MODE != 2 && threadIdx.x < 9) {
    float s = 0.f;
    for (int c = 0; c < C; ++c) s += __bfloat162float(Kp[c * 9 + threadIdx.x]);
    kb[threadIdx.x] = s / C;
  }
  for (int e = threadIdx.x; e < 2 * S; e += blockDim.x) buf0[e] = __float2bfloat16_rn(0.f);   // borders stay 0
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the zero fill before the async (bulk) writes
  __syncthreads();
  const uint32_t f0 = (uint32_t)__cvta_generic_to_shared(&full[0]), f1 = (uint32_t)__cvta_generic_to_shared(&full[1]);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf0);
  const uint32_t bytes = (uint32_t)m * d * 2;
  // one thread issues the sample's single bulk copy into rows 1..m
  auto issue = [&](int b, int s, uint32_t fb) {
    mbar_expect(fb, bytes);
    bulk_g2s(sb + (uint32_t)(s * S + P) * 2, img + (int64_t)b * m * d, bytes, fb);
  };
  if (threadIdx.x == 0) {
    mbar_init1(f0, 1);
    mbar_init1(f1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < B) issue(blockIdx.x, 0, f0);
  const int TPR = d / 4, groups = (int)blockDim.x / TPR, rg = threadIdx.x / TPR;
  const int c0 = (threadIdx.x % TPR) * 4;   // this thread's 4 output columns
  const int rpg = (m + groups - 1) / groups, i0 = rg * rpg, i1 = min(m, i0 + rpg);
  float wacc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) wacc[q] = 0.f;
  float kf[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) kf[q] = MODE == 0 ? kb[q] : MODE == 1 ? kb[8 - q] : 0.f;   // dgrad: flipped
  int it = 0;
  for (int b = blockIdx.x; b < B; b += gridDim.x, ++it) {
    const int s = it & 1;
    if (threadIdx.x == 0 && b + (int)gridDim.x < B) issue(b + gridDim.x, s ^ 1, s ? f0 : f1);   // next sample
    mbar_wait1(s ? f1 : f0, (it >> 1) & 1);
    if (rg < groups && i0 < i1) {
      const __nv_bfloat16* Sb = buf0 + s * S + c0;   // column c0 of padded row 0
      const bool lft = c0 > 0, rgt = c0 + 4 < d;
      // window: 3 rows x 6 columns (c0 - 1 .. c0 + 4) from three 8-B loads per row
      auto load_row = [&](int r, float* o6) {
        const uint2 a = lft ? *reinterpret_cast<const uint2*>(Sb + r * P - 4) : make_uint2(0u, 0u);
        const uint2 bq = *reinterpret_cast<const uint2*>(Sb + r * P);
        const uint2 c = rgt ? *reinterpret_cast<const uint2*>(Sb + r * P + 4) : make_uint2(0u, 0u);
        o6[0] = __uint_as_float(a.y & 0xffff0000u);   // column c0 - 1
        o6[1] = __uint_as_float(bq.x << 16); o6[2] = __uint_as_float(bq.x & 0xffff0000u);
        o6[3] = __uint_as_float(bq.y << 16); o6[4] = __uint_as_float(bq.y & 0xffff0000u);
        o6[5] = __uint_as_float(c.x << 16);            // column c0 + 4
      };
      float w[3][6];
      load_row(i0, w[1]);
      load_row(i0 + 1, w[2]);
      const int64_t base = (int64_t)b * m * d + c0;
      // wgrad: the dT rows of the next group of 8 are loaded while this group is combined (two groups in flight)
      uint2 gnext[MODE == 2 ? 8 : 1];
      if (MODE == 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          gnext[u] = (i0 + u < i1) ? __ldcs(reinterpret_cast<const uint2*>(other + base + (int64_t)(i0 + u) * d)) : make_uint2(0u, 0u);
      }
      for (int i = i0; i < i1; i += 8) {
        uint2 g8[8];
        if (MODE == 2) {
#pragma unroll
          for (int u = 0; u < 8; ++u) g8[u] = gnext[u];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            gnext[u] = (i + 8 + u < i1) ? __ldcs(reinterpret_cast<const uint2*>(other + base + (int64_t)(i + 8 + u) * d))
                                        : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ii = i + u;
          if (ii >= i1) break;
#pragma unroll
          for (int e = 0; e < 6; ++e) { w[0][e] = w[1][e]; w[1][e] = w[2][e]; }
          load_row(ii + 2, w[2]);
          if (MODE == 2) {
            const float g[4] = {__uint_as_float(g8[u].x << 16), __uint_as_float(g8[u].x & 0xffff0000u),
                                __uint_as_float(g8[u].y << 16), __uint_as_float(g8[u].y & 0xffff0000u)};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int e = 0; e < 3; ++e)
#pragma unroll
                for (int t = 0; t < 4; ++t) wacc[a * 3 + e] += g[t] * w[a][t + e];
          } else {
            float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int e = 0; e < 3; ++e)
#pragma unroll
                for (int t = 0; t < 4; ++t) o[t] += kf[a * 3 + e] * w[a][t + e];
            const int64_t off = base + (int64_t)ii * d;
            if (MODE == 0) {
              __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
              *reinterpret_cast<uint2*>(outT + off) = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
            } else {
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(outAcc + off), "f"(o[0]), "f"(o[1]), "f"(o[2]), "f"(o[3]) : "memory");
            }
          }
        }
      }
    }
    __syncthreads();   // every thread is done with buffer s before it is refilled (two samples ahead)
  }
  if (MODE == 2) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x / 32;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const float v = warp_sum(wacc[q]);
      if (lane == 0) red[q][wi] = v;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
      float v = 0.f;
      for (int ww = 0; ww < (int)(blockDim.x / 32); ++ww) v += red[threadIdx.x][ww];
      part[(int64_t)blockIdx.x * 9 + threadIdx.x] = v;
    }
  }
}
static bool conv_db_ok(int k, int m, int d, int dt, int pdt) {
  return k == 3 && dt == BF16 && pdt == BF16 && d % 8 == 0 && d <= 2048 && 2048 % d == 0 && (int64_t)m * d * 2 < (1 << 20) &&
         (size_t)2 * (m + 2) * d * 2 <= 200 * 1024;
}
template <int MODE>
static cudaError_t conv_db_launch(const void* img, const void* other, const void* Kp, int C, int B, int m, int d,
                                  void* outT, float* outAcc, float* part, int* grid_out, cudaStream_t st) {
  const size_t sm = (size_t)2 * (m + 2) * d * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_db_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  static int sms = 0;
  if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
  const int grid = std::min(B, sms);
  if (grid_out) *grid_out = grid;
  pdl_launch(conv_db_k<MODE>, grid, 512, sm, st, (const __nv_bfloat16*)img, (const __nv_bfloat16*)other,
                                         (const __nv_bfloat16*)Kp, C, B, m, d, (__nv_bfloat16*)outT, outAcc, part);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ conv (folded channel mean)
constexpr int CONV_MAXK = 7;
__device__ void load_kbar(const void* K, int pdt, int C, int k, float* kb) {
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < C; ++c) s += ld_as_f32(K, (int64_t)c * k * k + t, pdt);
    kb[t] = s / C;
  }
  __syncthreads();
}
__global__ void conv_fwd_k(const void* X, const void* K, int pdt, int C, int k, int B, int m, int d, void* T, int dt) {
  pdl_entry();
  __shared__ float kb[CONV_MAXK * CONV_MAXK];
  load_kbar(K, pdt, C, k, kb);
  const int r = (k - 1) / 2;
  int64_t total = (int64_t)B * m * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / ((int64_t)m * d);
    int i = (int)((t / d) % m), j = (int)(t % d);
    float s = 0.f;
    for (int a = 0; a < k; ++a) {
      int ii = i + a - r;
      if (ii < 0 || ii >= m) continue;
      for (int e = 0; e < k; ++e) {
        int jj = j + e - r;
        if (jj < 0 || jj >= d) continue;
        s += kb[a * k + e] * ld_as_f32(X, (b * m + ii) * d + jj, dt);
      }
    }
    st_from_f32(T, t, dt, s);
  }
}
cudaError_t conv_fwd(const void* X, const void* K, int pdt, int C, int k, int B, int m, int d, void* T, int dt,
                     cudaStream_t st) {
  if (k > CONV_MAXK) return cudaErrorInvalidValue;
  if (conv_db_ok(k, m, d, dt, pdt)) return conv_db_launch<0>(X, nullptr, K, C, B, m, d, T, nullptr, nullptr, nullptr, st);
  if (conv_sample_ok(k, m, d, dt == BF16 ? 2 : 4) && pdt == dt) {
    const int grid = std::min(B, 148 * 2);
    if (dt == BF16) return conv_sample_launch<__nv_bfloat16, 3, 0>(X, nullptr, K, C, B, m, d, T, nullptr, nullptr, grid, st);
    return conv_sample_launch<float, 3, 0>(X, nullptr, K, C, B, m, d, T, nullptr, nullptr, grid, st);
  }
  if (conv_band_ok(k, d, B) && pdt == dt) {
    if (dt == BF16) return k == 3 ? conv_band_launch<__nv_bfloat16, 3>(X, K, C, B, m, d, T, nullptr, false, st)
                                  : conv_band_launch<__nv_bfloat16, 5>(X, K, C, B, m, d, T, nullptr, false, st);
    return k == 3 ? conv_band_launch<float, 3>(X, K, C, B, m, d, T, nullptr, false, st)
                  : conv_band_launch<float, 5>(X, K, C, B, m, d, T, nullptr, false, st);
  }
  pdl_launch(conv_fwd_k, nblocks((int64_t)B * m * d), 256, 0, st, X, K, pdt, C, k, B, m, d, T, dt);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void conv_dgrad_k(const void* dT, const void* K, int pdt, int C, int k, int B, int m, int d, float* acc,
                             int dt) {
  pdl_entry();
  __shared__ float kb[CONV_MAXK * CONV_MAXK];
  load_kbar(K, pdt, C, k, kb);
  const int r = (k - 1) / 2;
  int64_t total = (int64_t)B * m * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / ((int64_t)m * d);
    int i = (int)((t / d) % m), j = (int)(t % d);
    float s = 0.f;
    for (int a = 0; a < k; ++a) {
      int ii = i - a + r;
      if (ii < 0 || ii >= m) continue;
      for (int e = 0; e < k; ++e) {
        int jj = j - e + r;
        if (jj < 0 || jj >= d) continue;
        s += kb[a * k + e] * ld_as_f32(dT, (b * m + ii) * d + jj, dt);
      }
    }
    acc[t] += s;
  }
}
cudaError_t conv_dgrad(const void* dT, const void* K, int pdt, int C, int k, int B, int m, int d, float* acc, int dt,
                       cudaStream_t st) {
  if (k > CONV_MAXK) return cudaErrorInvalidValue;
  if (conv_db_ok(k, m, d, dt, pdt)) return conv_db_launch<1>(dT, nullptr, K, C, B, m, d, nullptr, acc, nullptr, nullptr, st);
  if (conv_sample_ok(k, m, d, dt == BF16 ? 2 : 4) && pdt == dt) {
    const int grid = std::min(B, 148 * 2);
    if (dt == BF16) return conv_sample_launch<__nv_bfloat16, 3, 1>(dT, nullptr, K, C, B, m, d, nullptr, acc, nullptr, grid, st);
    return conv_sample_launch<float, 3, 1>(dT, nullptr, K, C, B, m, d, nullptr, acc, nullptr, grid, st);
  }
  if (conv_band_ok(k, d, B) && pdt == dt) {
    if (dt == BF16) return k == 3 ? conv_band_launch<__nv_bfloat16, 3>(dT, K, C, B, m, d, nullptr, acc, true, st)
                                  : conv_band_launch<__nv_bfloat16, 5>(dT, K, C, B, m, d, nullptr, acc, true, st);
    return k == 3 ? conv_band_launch<float, 3>(dT, K, C, B, m, d, nullptr, acc, true, st)
                  : conv_band_launch<float, 5>(dT, K, C, B, m, d, nullptr, acc, true, st);
  }
  pdl_launch(conv_dgrad_k, nblocks((int64_t)B * m * d), 256, 0, st, dT, K, pdt, C, k, B, m, d, acc, dt);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void conv_wgrad_k(const void* dT, const void* X, int k, int B, int m, int d, int dt, float* part,
                             int64_t per_block) {
  pdl_entry();
  __shared__ float red[CONV_MAXK * CONV_MAXK][8];
  const int r = (k - 1) / 2;
  float s[CONV_MAXK * CONV_MAXK];
  for (int q = 0; q < k * k; ++q) s[q] = 0.f;
  int64_t total = (int64_t)B * m * d;
  int64_t t0 = blockIdx.x * per_block, t1 = min(total, t0 + per_block);
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    int64_t b = t / ((int64_t)m * d);
    int i = (int)((t / d) % m), j = (int)(t % d);
    float g = ld_as_f32(dT, t, dt);
    for (int a = 0; a < k; ++a) {
      int ii = i + a - r;
      if (ii < 0 || ii >= m) continue;
      for (int e = 0; e < k; ++e) {
        int jj = j + e - r;
        if (jj < 0 || jj >= d) continue;
        s[a * k + e] += g * ld_as_f32(X, (b * m + ii) * d + jj, dt);
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  for (int q = 0; q < k * k; ++q) {
    float v = warp_sum(s[q]);
    if (lane == 0) red[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < k * k) {
    float v = 0.f;
    for (int ww = 0; ww < (int)(blockDim.x / 32); ++ww) v += red[threadIdx.x][ww];
    part[(int64_t)blockIdx.x * k * k + threadIdx.x] = v;
  }
}
__global__ void conv_wgrad_fin_k(const float* part, int nparts, int C, int kk, float* dK) {
  pdl_entry();
  for (int t = threadIdx.x; t < kk; t += blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * kk + t];
    s /= C;
    for (int c = 0; c < C; ++c) dK[c * kk + t] += s;    // identical for every channel (R12)
  }
}
cudaError_t conv_wgrad(const void* dT, const void* X, int C, int k, int B, int m, int d, int dt, float* dK,
                       float* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (k > CONV_MAXK) return cudaErrorInvalidValue;
  if (conv_db_ok(k, m, d, dt, dt) && (size_t)std::min(B, 148) * 9 * sizeof(float) <= scratch_bytes) {
    int grid = 0;
    cudaError_t e = conv_db_launch<2>(X, dT, nullptr, C, B, m, d, nullptr, nullptr, scratch, &grid, st);
    if (e != cudaSuccess) return e;
    pdl_launch(conv_wgrad_fin_k, 1, 64, 0, st, scratch, grid, C, k * k, dK);
    ++g_launches;
    return cudaGetLastError();
  }
  if (conv_sample_ok(k, m, d, dt == BF16 ? 2 : 4)) {
    const int grid = std::min(B, 148 * 2);
    if ((size_t)grid * k * k * sizeof(float) <= scratch_bytes) {
      cudaError_t e = dt == BF16 ? conv_sample_launch<__nv_bfloat16, 3, 2>(X, dT, nullptr, C, B, m, d, nullptr, nullptr, scratch, grid, st)
                                 : conv_sample_launch<float, 3, 2>(X, dT, nullptr, C, B, m, d, nullptr, nullptr, scratch, grid, st);
      if (e != cudaSuccess) return e;
      pdl_launch(conv_wgrad_fin_k, 1, 64, 0, st, scratch, grid, C, k * k, dK);
      ++g_launches;
      return cudaGetLastError();
    }
  }
  const int64_t bands = (int64_t)((m + CV_RB - 1) / CV_RB) * B;
  const int grid = (int)std::min<int64_t>(bands, 148 * 4);
  if (conv_band_ok(k, d, B) && (size_t)grid * k * k * sizeof(float) <= scratch_bytes) {
    const int R = (k - 1) / 2;
    const size_t sm = (size_t)(CV_RB + 2 * R) * (d + 2 * R) * sizeof(float);
    if (dt == BF16) {
      if (k == 3) pdl_launch(conv_wgrad_band_k<__nv_bfloat16, 3>, grid, 256, sm, st, (const __nv_bfloat16*)dT, (const __nv_bfloat16*)X, m, d, scratch, B);
      else pdl_launch(conv_wgrad_band_k<__nv_bfloat16, 5>, grid, 256, sm, st, (const __nv_bfloat16*)dT, (const __nv_bfloat16*)X, m, d, scratch, B);
    } else {
      if (k == 3) pdl_launch(conv_wgrad_band_k<float, 3>, grid, 256, sm, st, (const float*)dT, (const float*)X, m, d, scratch, B);
      else pdl_launch(conv_wgrad_band_k<float, 5>, grid, 256, sm, st, (const float*)dT, (const float*)X, m, d, scratch, B);
    }
    pdl_launch(conv_wgrad_fin_k, 1, 64, 0, st, scratch, grid, C, k * k, dK);
    g_launches += 2;
    return cudaGetLastError();
  }
  int64_t total = (int64_t)B * m * d;
  int nb = (int)std::min<int64_t>(std::max<int64_t>(1, total / 4096), 148 * 4);
  nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * k * k)));
  int64_t per = (total + nb - 1) / nb;
  nb = (int)((total + per - 1) / per);
  pdl_launch(conv_wgrad_k, nb, 256, 0, st, dT, X, k, B, m, d, dt, scratch, per);
  pdl_launch(conv_wgrad_fin_k, 1, 64, 0, st, scratch, nb, C, k * k, dK);
  g_launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ head + loss
// One block per sample.  Pooling: thread (ry, cx) sums rows ry, ry + RY, ... of column chunk cx (VEC
// consecutive columns), then the RY partials are added in fixed order.  dY[b] = (dz_b / m) w broadcast.
template <int VEC>
__global__ void __launch_bounds__(256) head_v(const __nv_bfloat16* __restrict__ Y, const __nv_bfloat16* __restrict__ w,
                                              const __nv_bfloat16* __restrict__ bh, const float* __restrict__ labels,
                                              int m, int d, int Bg, __nv_bfloat16* __restrict__ dY, float* pooled,
                                              float* z, float* lossb, float* dz, int do_bwd, float* __restrict__ hpart) {
  pdl_entry();
  extern __shared__ float hs[];   // [RY][d] partial column sums
  __shared__ float red[8];
  __shared__ float dzs;
  const int b = blockIdx.x;
  const int CX = d / VEC, RY = blockDim.x / CX;
  const int cx = threadIdx.x % CX, ry = threadIdx.x / CX;
  const __nv_bfloat16* Yb = Y + (int64_t)b * m * d;
  if (ry < RY) {
    float a[VEC];
#pragma unroll
    for (int t = 0; t < VEC; ++t) a[t] = 0.f;
    for (int r = ry; r < m; r += RY) {
      const uint4 u = *reinterpret_cast<const uint4*>(Yb + (int64_t)r * d + cx * VEC);
      const uint32_t q[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) { a[2 * t] += __uint_as_float(q[t] << 16); a[2 * t + 1] += __uint_as_float(q[t] & 0xffff0000u); }
    }
#pragma unroll
    for (int t = 0; t < VEC; ++t) hs[ry * d + cx * VEC + t] = a[t];
  }
  __syncthreads();
  float part = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < RY; ++k) s += hs[k * d + c];
    s /= m;
    pooled[(int64_t)b * d + c] = s;
    part += s * __bfloat162float(w[c]);
  }
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) s += red[q];
    const float zz = s + __bfloat162float(bh[0]);
    z[b] = zz;
    if (do_bwd) {
      const float y = labels[b];
      lossb[b] = fmaxf(zz, 0.f) - y * zz + log1pf(expf(-fabsf(zz)));
      const float sg = 1.f / (1.f + expf(-zz));
      dzs = (sg - y) / (float)Bg;
      dz[b] = dzs;
    }
  }
  __syncthreads();
  if (!do_bwd) return;
  if (hpart) {   // this sample's row of the head-gradient / loss partials: [dz pooled (d), dz, loss]
    for (int c = threadIdx.x; c < d; c += blockDim.x) hpart[(int64_t)b * (d + 2) + c] = dzs * pooled[(int64_t)b * d + c];
    if (threadIdx.x == 0) { hpart[(int64_t)b * (d + 2) + d] = dzs; hpart[(int64_t)b * (d + 2) + d + 1] = lossb[b]; }
  }
  if (!dY) return;   // dY formed by the last layer's LayerNorm backward instead (ln_bwd vdz)
  const float g = dzs / m;
  // every row of dY[b] is the same vector g * w
  for (int q = threadIdx.x; q < m * CX; q += blockDim.x) {
    const int r = q / CX, c0 = (q - r * CX) * VEC;
    const uint4 wu = *reinterpret_cast<const uint4*>(w + c0);
    const uint32_t wq[4] = {wu.x, wu.y, wu.z, wu.w};
    uint32_t o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(g * __uint_as_float(wq[t] << 16), g * __uint_as_float(wq[t] & 0xffff0000u));
      o[t] = *reinterpret_cast<uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>(dY + (int64_t)b * m * d + (int64_t)r * d + c0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}
__global__ void head_k(const void* Y, const void* w, const void* bh, int pdt, const float* labels, int m, int d, int Bg,
                       void* dY, int dt, float* pooled, float* z, float* lossb, float* dz, int do_bwd) {
  pdl_entry();
  __shared__ float red[32];
  const int b = blockIdx.x;
  float part = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int t = 0; t < m; ++t) s += ld_as_f32(Y, ((int64_t)b * m + t) * d + c, dt);
    s /= m;
    pooled[(int64_t)b * d + c] = s;
    part += s * ld_as_f32(w, c, pdt);
  }
  part = warp_sum(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = part;
  __syncthreads();
  __shared__ float dzs;
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) s += red[q];
    float zz = s + ld_as_f32(bh, 0, pdt);
    z[b] = zz;
    if (do_bwd) {
      float y = labels[b];
      lossb[b] = fmaxf(zz, 0.f) - y * zz + log1pf(expf(-fabsf(zz)));
      float sg = 1.f / (1.f + expf(-zz));
      dzs = (sg - y) / (float)Bg;
      dz[b] = dzs;
    }
  }
  __syncthreads();
  if (!do_bwd) return;
  const float g = dzs / m;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += blockDim.x) {
    int c = (int)(e % d);
    st_from_f32(dY, (int64_t)b * m * d + e, dt, g * ld_as_f32(w, c, pdt));
  }
}
// two-pass deterministic reduction of the head gradients over samples:
// part[blk] = (sum_b dz_b pooled_b[0..d), sum_b dz_b, sum_b loss_b) over the block's sample chunk
__global__ void head_part_k(const float* pooled, const float* dz, const float* lossb, int B, int d, int per,
                            float* part) {
  pdl_entry();
  const int b0 = blockIdx.x * per, b1 = min(B, b0 + per);
  for (int c = threadIdx.x; c < d + 2; c += blockDim.x) {
    float s = 0.f;
    for (int b = b0; b < b1; ++b) {
      s += c < d ? dz[b] * pooled[(int64_t)b * d + c] : (c == d ? dz[b] : lossb[b]);
    }
    part[(int64_t)blockIdx.x * (d + 2) + c] = s;
  }
}
cudaError_t head_fwd_bwd(const void* Y, const void* w, const void* bh, int pdt, const float* labels, int B, int m, int d,
                         int Bg, void* dY, int dt, float* pooled, float* z, float* lossb, float* dz, float* loss_out,
                         float* dw, float* db, int do_bwd, cudaStream_t st, cudaStream_t st_red,
                         cudaEvent_t ev_red) {
  if (dt == BF16 && pdt == BF16 && d % 8 == 0 && d / 8 <= 256 && ((uintptr_t)Y % 16) == 0 && ((uintptr_t)w % 16) == 0 &&
      (!do_bwd || ((uintptr_t)dY % 16) == 0)) {
    const int RY = 256 / (d / 8);
    float* hpart = pooled + (int64_t)B * d;   // [B][d + 2] (sized by the runtime)
    pdl_launch(head_v<8>, B, 256, (size_t)RY * d * sizeof(float), st, (const __nv_bfloat16*)Y, (const __nv_bfloat16*)w,
        (const __nv_bfloat16*)bh, labels, m, d, Bg, (__nv_bfloat16*)dY, pooled, z, lossb, dz, do_bwd,
        do_bwd ? hpart : nullptr);
    ++g_launches;
    if (do_bwd) {
      cudaStream_t sr = st;
      if (st_red && ev_red && st_red != st) {   // dY is what st needs next; the head sums can trail
        cudaEventRecord(ev_red, st);
        cudaStreamWaitEvent(st_red, ev_red, 0);
        sr = st_red;
      }
      part_sum(hpart, B, d + 2, dw, d, db, 1, loss_out, 1.f / (float)Bg, sr);   // fixed order over samples
    }
    return cudaGetLastError();
  } else {
    pdl_launch(head_k, B, 256, 0, st, Y, w, bh, pdt, labels, m, d, Bg, dY, dt, pooled, z, lossb, dz, do_bwd);
  }
  ++g_launches;
  if (do_bwd) {
    const int per = 32, nparts = (B + per - 1) / per;
    float* part = pooled + (int64_t)B * d;   // scratch after pooled (sized by the runtime)
    pdl_launch(head_part_k, nparts, 128, 0, st, pooled, dz, lossb, B, d, per, part);
    ++g_launches;
    part_sum(part, nparts, d + 2, dw, d, db, 1, loss_out, 1.f / (float)Bg, st);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ block-diagonal token map
// out[i][k] (bf16, [spt m][spt l]) = W[i % m][k % l] if i / m == k / l else 0; W bf16 [m][l]
__global__ void blockdiag_k(const __nv_bfloat16* W, int m, int l, int spt, __nv_bfloat16* out) {
  pdl_entry();
  const int n = spt * m * spt * l;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = t / (spt * l), k = t - i * (spt * l);
    out[t] = (i / m == k / l) ? W[(i % m) * l + (k % l)] : __float2bfloat16_rn(0.f);
  }
}
cudaError_t blockdiag(const void* W, int m, int l, int spt, void* out, cudaStream_t st) {
  const int n = spt * m * spt * l;
  pdl_launch(blockdiag_k, (n + 255) / 256, 256, 0, st, (const __nv_bfloat16*)W, m, l, spt, (__nv_bfloat16*)out);
  ++g_launches;
  return cudaGetLastError();
}

// out[i][k] (bf16, [spt l][spt m]) = W[k % m][i % l] if i / l == k / m else 0: blockdiag(W^T, .., W^T)
__global__ void blockdiag_t_k(const __nv_bfloat16* W, int m, int l, int spt, __nv_bfloat16* out) {
  pdl_entry();
  const int n = spt * l * spt * m;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = t / (spt * m), k = t - i * (spt * m);
    out[t] = (i / l == k / m) ? W[(k % m) * l + (i % l)] : __float2bfloat16_rn(0.f);
  }
}
cudaError_t blockdiag_t(const void* W, int m, int l, int spt, void* out, cudaStream_t st) {
  const int n = spt * l * spt * m;
  pdl_launch(blockdiag_t_k, (n + 255) / 256, 256, 0, st, (const __nv_bfloat16*)W, m, l, spt, (__nv_bfloat16*)out);
  ++g_launches;
  return cudaGetLastError();
}

// All of a step's block-diagonal token maps in one launch (blockIdx.y = job): jobs with tr = 1 build
// blockdiag_t (the forward's packed token projection), tr = 0 blockdiag (the DCN backward's packed dT).
__global__ void blockdiag_multi_k(BdJobs jobs) {
  pdl_entry();
  const BdJob& j = jobs.job[blockIdx.y];
  const int m = j.m, l = j.l, spt = j.spt;
  const int n = spt * m * spt * l;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    __nv_bfloat16 v = __float2bfloat16_rn(0.f);
    if (j.tr) {
      const int i = t / (spt * m), k = t - i * (spt * m);
      if (i / l == k / m) v = j.W[(k % m) * l + (i % l)];
    } else {
      const int i = t / (spt * l), k = t - i * (spt * l);
      if (i / m == k / l) v = j.W[(i % m) * l + (k % l)];
    }
    j.out[t] = v;
  }
}
cudaError_t blockdiag_multi(const BdJobs& jobs, cudaStream_t st) {
  if (jobs.n <= 0) return cudaSuccess;
  pdl_launch(blockdiag_multi_k, dim3(64, jobs.n), 256, 0, st, jobs);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ SGD, casts, init
__global__ void sgd_cast_k(float* master, const float* grad, float lr, void* copy, int dt, int64_t n) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    float v = master[t];
    if (grad) { v -= lr * grad[t]; master[t] = v; }
    if (copy) st_from_f32(copy, t, dt, v);
  }
}
// 4 elements per thread (n % 4 == 0, 16-B aligned fp32 arrays, 8-B aligned bf16 copy)
__global__ void sgd_cast4_k(float4* __restrict__ master, const float4* __restrict__ grad, float lr, uint2* __restrict__ copy,
                            int64_t n4) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
    float4 v = master[t];
    if (grad) {
      const float4 g = grad[t];
      v.x -= lr * g.x; v.y -= lr * g.y; v.z -= lr * g.z; v.w -= lr * g.w;
      master[t] = v;
    }
    if (copy) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
      copy[t] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
  }
}
cudaError_t sgd_cast(float* master, const float* grad, float lr, void* copy, int dt, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n % 4 == 0 && (!copy || dt == BF16) && ((uintptr_t)master % 16) == 0 && ((uintptr_t)grad % 16) == 0 &&
      ((uintptr_t)copy % 8) == 0) {
    pdl_launch(sgd_cast4_k, nblocks(n / 4, 256, 148 * 16), 256, 0, st, (float4*)master, (const float4*)grad, lr, (uint2*)copy, n / 4);
  } else {
    pdl_launch(sgd_cast_k, nblocks(n), 256, 0, st, master, grad, lr, copy, dt, n);
  }
  ++g_launches;
  return cudaGetLastError();
}
// Multi-tensor SGD: every parameter group of the step in ONE launch (segments concatenated in 4-element units)
__global__ void __launch_bounds__(256) sgd_multi_k(SgdSegs segs, float lr) {
  pdl_entry();
  int64_t tot = 0;
  for (int s = 0; s < segs.n; ++s) tot += segs.n4[s];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    int64_t u = t;
    while (u >= segs.n4[s]) { u -= segs.n4[s]; ++s; }
    float4* master = reinterpret_cast<float4*>(segs.master[s]);
    float4 v = master[u];
    const float4 g = reinterpret_cast<const float4*>(segs.grad[s])[u];
    v.x -= lr * g.x; v.y -= lr * g.y; v.z -= lr * g.z; v.w -= lr * g.w;
    master[u] = v;
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<uint2*>(segs.copy[s])[u] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}
// Adam on the fp32 master shard; the moments are stored in MT (fp32, or bf16 for the BF16 optimizer of R35:
// each step computes in fp32 from the stored moments, updates theta with the fp32 values and stores them RNE)
template <typename MT>
__global__ void __launch_bounds__(256) adam_k(float* __restrict__ master, const float* __restrict__ grad,
                                             MT* __restrict__ m, MT* __restrict__ v, void* copy, int dt, int64_t n,
                                             float lr, float b1, float b2, float eps, const int* __restrict__ step) {
  pdl_entry();
  const float t = (float)(*step + 1);
  const float c1 = 1.f - powf(b1, t), c2 = 1.f - powf(b2, t);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float g = grad[i];
    const float mi = b1 * (float)m[i] + (1.f - b1) * g;
    const float vi = b2 * (float)v[i] + (1.f - b2) * g * g;
    m[i] = (MT)mi;
    v[i] = (MT)vi;
    const float p = master[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    master[i] = p;
    st_from_f32(copy, i, dt, p);
  }
}
__global__ void adam_count_k(int* step) {
  pdl_entry();
  if (threadIdx.x == 0 && blockIdx.x == 0) *step += 1;
}
cudaError_t adam_step(float* master, const float* grad, void* m, void* v, int mdt, void* copy, int dt, int64_t n, float lr,
                      float b1, float b2, float eps, const int* step, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (mdt == BF16)
    pdl_launch(adam_k<__nv_bfloat16>, nblocks(n, 256, 148 * 16), 256, 0, st, master, grad, (__nv_bfloat16*)m,
               (__nv_bfloat16*)v, copy, dt, n, lr, b1, b2, eps, step);
  else
    pdl_launch(adam_k<float>, nblocks(n, 256, 148 * 16), 256, 0, st, master, grad, (float*)m, (float*)v, copy, dt, n, lr,
               b1, b2, eps, step);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t adam_count(int* step, cudaStream_t st) {
  pdl_launch(adam_count_k, 1, 32, 0, st, step);
  ++g_launches;
  return cudaGetLastError();
}
// ------------------------------------------------------------------ sum / weighted-sum ensembles (R27)
// one warp per row; lane holds columns lane, lane + 32, ... (d <= 1024)
__global__ void __launch_bounds__(256) ens_ln_fwd_k(EnsU U, const void* w, int pdt, const float* base32, const void* basex,
                                                    const void* gamma, const void* beta, float eps, int64_t rows, int d,
                                                    void* Y, void* R, float* mu, float* rstd, int dt) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  float wk[16];
  for (int i = 0; i < U.k; ++i) wk[i] = w ? ld_as_f32(w, i, pdt) : 1.f;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    float v[32];
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int c = lane + 32 * q;
      v[q] = 0.f;
      if (c < d) {
        const int64_t o = r * d + c;
        float a = base32 ? base32[o] : ld_as_f32(basex, o, dt);
        for (int i = 0; i < U.k; ++i) a += wk[i] * U.u[i][o];
        v[q] = a;
        s += a;
      }
    }
    const float mean = warp_sum(s) / d;
    float s2 = 0.f;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (lane + 32 * q < d) { const float t = v[q] - mean; s2 += t * t; }
    const float rs = rsqrtf(warp_sum(s2) / d + eps);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int c = lane + 32 * q;
      if (c < d) {
        const int64_t o = r * d + c;
        st_from_f32(R, o, dt, v[q]);
        st_from_f32(Y, o, dt, (v[q] - mean) * rs * ld_as_f32(gamma, c, dt) + ld_as_f32(beta, c, dt));
      }
    }
    if (lane == 0) { mu[r] = mean; rstd[r] = rs; }
  }
}
cudaError_t ens_ln_fwd(const EnsU& U, const void* w, int pdt, const float* base32, const void* basex, const void* gamma,
                       const void* beta, float eps, int64_t rows, int d, void* Y, void* R, float* mu, float* rstd, int dt,
                       cudaStream_t st) {
  if (d > 1024 || U.k < 1 || U.k > 16 || (!base32 && !basex)) return cudaErrorInvalidValue;
  pdl_launch(ens_ln_fwd_k, nblocks(rows, 8, 148 * 64), 256, 0, st, U, w, pdt, base32, basex, gamma, beta, eps, rows, d, Y, R,
             mu, rstd, dt);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void ens_scale_k(const void* dR, const void* w, int i, int pdt, void* out, int64_t n, int dt) {
  pdl_entry();
  const float a = ld_as_f32(w, i, pdt);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    st_from_f32(out, t, dt, a * ld_as_f32(dR, t, dt));
}
cudaError_t ens_scale(const void* dR, const void* w, int i, int pdt, void* out, int64_t n, int dt, cudaStream_t st) {
  pdl_launch(ens_scale_k, nblocks(n), 256, 0, st, dR, w, i, pdt, out, n, dt);
  ++g_launches;
  return cudaGetLastError();
}
constexpr int ENS_DOT_BLOCKS = 592;
__global__ void __launch_bounds__(256) ens_dot_k(const float* U, const void* dR, int dt, int64_t n, float* part) {
  pdl_entry();
  float s = 0.f;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    s += U[t] * ld_as_f32(dR, t, dt);
  __shared__ float red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int q = 0; q < 8; ++q) a += red[q];
    part[blockIdx.x] = a;
  }
}
__global__ void ens_dot_fin_k(const float* part, int np, float* acc) {
  pdl_entry();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float a = 0.f;
    for (int q = 0; q < np; ++q) a += part[q];
    *acc += a;
  }
}
cudaError_t ens_dot(const float* U, const void* dR, int dt, int64_t n, float* acc, float* scratch, cudaStream_t st) {
  pdl_launch(ens_dot_k, ENS_DOT_BLOCKS, 256, 0, st, U, dR, dt, n, scratch);
  pdl_launch(ens_dot_fin_k, 1, 32, 0, st, (const float*)scratch, ENS_DOT_BLOCKS, acc);
  g_launches += 2;
  return cudaGetLastError();
}
// S = dG + dG^T per sample (32 x 32 tiles through shared memory: both reads coalesced)
__global__ void sym_add_k(const float* __restrict__ dG, void* S, int dt, int d) {
  pdl_entry();
  __shared__ float tl[32][33];
  const int64_t base = (int64_t)blockIdx.z * d * d;
  const int c0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)   // tile (k0.., c0..) transposed into tl[c][k]
    if (k0 + r < d && c0 + threadIdx.x < d) tl[threadIdx.x][r] = dG[base + (int64_t)(k0 + r) * d + c0 + threadIdx.x];
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c0 + r, k = k0 + threadIdx.x;
    if (c < d && k < d) st_from_f32(S, base + (int64_t)c * d + k, dt, dG[base + (int64_t)c * d + k] + tl[r][threadIdx.x]);
  }
}
cudaError_t sym_add(const float* dG, void* S, int dt, int B, int d, cudaStream_t st) {
  pdl_launch(sym_add_k, dim3((d + 31) / 32, (d + 31) / 32, B), dim3(32, 8), 0, st, dG, S, dt, d);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t sgd_multi(const SgdSegs& segs, float lr, cudaStream_t st) {
  int64_t tot = 0;
  for (int s = 0; s < segs.n; ++s) {
    if ((uintptr_t)segs.master[s] % 16 || (uintptr_t)segs.grad[s] % 16 || (uintptr_t)segs.copy[s] % 8)
      return cudaErrorInvalidValue;
    tot += segs.n4[s];
  }
  if (tot == 0) return cudaSuccess;
  pdl_launch(sgd_multi_k, nblocks(tot, 256, 148 * 16), 256, 0, st, segs, lr);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void cast_k(const void* src, int sdt, void* dst, int ddt, int64_t n) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    st_from_f32(dst, t, ddt, ld_as_f32(src, t, sdt));
}
// fp32 -> bf16, 8 elements per thread
__global__ void cast8_k(const float4* __restrict__ src, uint4* __restrict__ dst, int64_t n8) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8; t += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = __ldcs(src + 2 * t), b = __ldcs(src + 2 * t + 1);
    __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
    dst[t] = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                        *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
  }
}
cudaError_t cast(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (sdt == F32 && ddt == BF16 && n % 8 == 0 && ((uintptr_t)src % 16) == 0 && ((uintptr_t)dst % 16) == 0)
    pdl_launch(cast8_k, nblocks(n / 8, 256, 148 * 16), 256, 0, st, (const float4*)src, (uint4*)dst, n / 8);
  else
    pdl_launch(cast_k, nblocks(n), 256, 0, st, src, sdt, dst, ddt, n);
  ++g_launches;
  return cudaGetLastError();
}
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void init_uniform_k(float* p, int64_t n, float bound, unsigned long long seed, unsigned long long sid,
                               int64_t idx0) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = splitmix64(seed ^ splitmix64(sid * 0x100000001B3ull + (unsigned long long)(idx0 + t)));
    float u = (float)((h >> 40) * (1.0 / 16777216.0));   // [0,1)
    p[t] = bound * (2.f * u - 1.f);
  }
}
cudaError_t init_uniform(float* p, int64_t n, float bound, unsigned long long seed, unsigned long long stream_id,
                         int64_t idx0, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(init_uniform_k, nblocks(n), 256, 0, st, p, n, bound, seed, stream_id, idx0);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void fill_k(float* p, int64_t n, float v) {
  pdl_entry();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) p[t] = v;
}
cudaError_t fill(float* p, int64_t n, float v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  pdl_launch(fill_k, nblocks(n), 256, 0, st, p, n, v);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace dhen

// ------------------------------------------------------------------ dense-token injection (R38, NEXT#3)
namespace dhen {
namespace {
template <typename T>
__global__ void inject_copy_k(const T* __restrict__ X, const T* __restrict__ X0, int64_t B, int mi, int nD, int m0,
                              int d4, T* __restrict__ Xin) {
  pdl_entry();
  const int mm = mi + nD;
  const int64_t n = B * mm * d4;   // 4-element groups
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / ((int64_t)mm * d4);
    const int64_t r = i - b * mm * d4;
    const int t = (int)(r / d4), c = (int)(r - (int64_t)t * d4);
    const T* src = t < mi ? X + ((b * mi + t) * d4 + c) * 4 : X0 + ((b * m0 + (t - mi)) * d4 + c) * 4;
    T* dst = Xin + i * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[k] = src[k];
  }
}
__global__ void inject_dD_k(const float* __restrict__ accm, int64_t B, int mi, int nD, int d, float* __restrict__ dD) {
  pdl_entry();
  const int64_t n = B * nD * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / ((int64_t)nD * d);
    const int64_t r = i - b * nD * d;
    dD[i] += accm[(b * (mi + nD)) * d + (int64_t)mi * d + r];
  }
}
template <typename T>
__global__ void inject_final_k(const float* __restrict__ acc_sc, const float* __restrict__ accm, int m_mod,
                               const float* __restrict__ dD, int nDadd, int64_t B, int mi, int d, T* __restrict__ dX) {
  pdl_entry();
  const int64_t n = B * mi * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / ((int64_t)mi * d);
    const int64_t r = i - b * mi * d;
    const int t = (int)(r / d);
    float v = acc_sc[i] + accm[b * (int64_t)m_mod * d + r];
    if (t < nDadd) v += dD[(b * nDadd + t) * d + (r - (int64_t)t * d)];
    dX[i] = fromf<T>(v);
  }
}
}  // namespace

cudaError_t inject_copy(const void* X, const void* X0, int dt, int64_t B, int mi, int nD, int m0, int d, void* Xin,
                        cudaStream_t st) {
  const int64_t n = B * (mi + nD) * (d / 4);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dt == BF16)
    pdl_launch(inject_copy_k<__nv_bfloat16>, grid, 256, 0, st, (const __nv_bfloat16*)X, (const __nv_bfloat16*)X0, B, mi, nD,
               m0, d / 4, (__nv_bfloat16*)Xin);
  else
    pdl_launch(inject_copy_k<float>, grid, 256, 0, st, (const float*)X, (const float*)X0, B, mi, nD, m0, d / 4, (float*)Xin);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t inject_dD(const float* accm, int64_t B, int mi, int nD, int d, float* dD, cudaStream_t st) {
  const int64_t n = B * nD * d;
  pdl_launch(inject_dD_k, (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st, accm, B, mi, nD, d, dD);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t inject_final(const float* acc_sc, const float* accm, int m_mod, const float* dD, int nDadd, int64_t B, int mi,
                         int d, void* dX, int dt, cudaStream_t st) {
  const int64_t n = B * mi * d;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (dt == BF16)
    pdl_launch(inject_final_k<__nv_bfloat16>, grid, 256, 0, st, acc_sc, accm, m_mod, dD, nDadd, B, mi, d, (__nv_bfloat16*)dX);
  else
    pdl_launch(inject_final_k<float>, grid, 256, 0, st, acc_sc, accm, m_mod, dD, nDadd, B, mi, d, (float*)dX);
  ++g_launches;
  return cudaGetLastError();
}
}  // namespace dhen
