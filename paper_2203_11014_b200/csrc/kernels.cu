// kernels.cu — memory-bound DHEN kernels: triangle gather/scatter (Dot), LayerNorm
// fwd/bwd, column sums, softmax fwd/bwd, DCN backward elementwise, 3x3 conv,
// head + BCE loss, SGD.  Warp-per-row reductions via shuffles; every cross-block
// reduction is a fixed-order two-pass (deterministic).
#include "kernels.h"
#include <algorithm>

namespace dhen {

static inline int nblocks(int64_t n, int per = 256, int cap = 148 * 32) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, cap));
}

// ------------------------------------------------------------------ Dot triangle
__global__ void triu_extract_k(const float* G, void* Z, int dt, int B, int m, int64_t ldz) {
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
  triu_extract_k<<<nblocks(total), 256, 0, st>>>(G, Z, dt, B, m, ldz);
  ++g_launches;
  return cudaGetLastError();
}

__global__ void sym_from_triu_k(const void* dZ, void* S, int dt, int B, int m, int64_t ldz) {
  int64_t total = (int64_t)B * m * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(t / ((int64_t)m * m));
    int r = (int)(t % ((int64_t)m * m));
    int i = r / m, j = r % m;
    float v = 0.f;
    if (i != j) {
      int a = min(i, j), c = max(i, j);
      int p = a * m - a * (a + 1) / 2 + (c - a - 1);
      v = ld_as_f32(dZ, (int64_t)b * ldz + p, dt);
    }
    st_from_f32(S, t, dt, v);
  }
}
cudaError_t sym_from_triu(const void* dZ, void* S, int dt, int B, int m, int64_t ldz, cudaStream_t st) {
  sym_from_triu_k<<<nblocks((int64_t)B * m * m), 256, 0, st>>>(dZ, S, dt, B, m, ldz);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ LayerNorm
constexpr int LN_MAXQ_ALL = 32;  // d <= 1024

template <int LN_MAXQ>
__global__ void ln_fwd_k(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                         int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt) {
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
cudaError_t ln_fwd(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                   int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt, cudaStream_t st) {
  if (d > 32 * LN_MAXQ_ALL) return cudaErrorInvalidValue;
  const int nb = nblocks(rows, 8, 148 * 64);
  if (d <= 128) ln_fwd_k<4><<<nb, 256, 0, st>>>(U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  else if (d <= 256) ln_fwd_k<8><<<nb, 256, 0, st>>>(U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  else ln_fwd_k<32><<<nb, 256, 0, st>>>(U, addx, gamma, beta, pdt, eps, rows, d, Y, Rsave, mu, rstd, dt);
  ++g_launches;
  return cudaGetLastError();
}

template <int LN_MAXQ>
__global__ void ln_bwd_k(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                         const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                         float* part, int64_t rows_per_block) {
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

__global__ void reduce_parts_k(const float* part, int nparts, int n, float* out0, float* out1) {
  // part [nparts][2n] -> out0 += sum part[:, :n], out1 += sum part[:, n:]
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < 2 * n; c += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * 2 * n + c];
    if (c < n) { if (out0) out0[c] += s; } else { if (out1) out1[c - n] += s; }
  }
}

cudaError_t ln_bwd(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                   const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                   float* dgamma, float* dbeta, float* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (d > 32 * LN_MAXQ_ALL) return cudaErrorInvalidValue;
  int nb = (int)std::min<int64_t>((rows + 63) / 64, 148 * 4);
  nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * 2 * d)));
  if (nb < 1) return cudaErrorInvalidValue;
  int64_t rpb = (rows + nb - 1) / nb;
  nb = (int)((rows + rpb - 1) / rpb);
  if (d <= 128)
    ln_bwd_k<4><<<nb, 256, 0, st>>>(dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  else if (d <= 256)
    ln_bwd_k<8><<<nb, 256, 0, st>>>(dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  else
    ln_bwd_k<32><<<nb, 256, 0, st>>>(dY, dydt, Rsave, mu, rstd, gamma, pdt, rows, d, dR, dt, acc, acc_mode, scratch, rpb);
  reduce_parts_k<<<nblocks(2 * d), 256, 0, st>>>(scratch, nb, d, dgamma, dbeta);
  g_launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ column sums
__global__ void colsum_part_k(const void* src, int dt, int64_t rows, int cols, int64_t ld, int64_t rpc, float* part) {
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
__global__ void colsum_fin_k(const float* part, int nparts, int cols, float* out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * cols + c];
    out[c] += s;
  }
}
cudaError_t colsum_add(const void* src, int dt, int64_t rows, int cols, int64_t ld, float* out, float* scratch,
                       size_t scratch_bytes, cudaStream_t st) {
  int cb = (cols + 31) / 32;
  int64_t nch = std::max<int64_t>(1, std::min<int64_t>(rows / 256, std::max(1, 296 / cb)));
  nch = std::min<int64_t>(nch, (int64_t)(scratch_bytes / (sizeof(float) * cols)));
  if (nch < 1) return cudaErrorInvalidValue;
  int64_t rpc = (rows + nch - 1) / nch;
  nch = (rows + rpc - 1) / rpc;
  if (nch < 1) nch = 1;
  colsum_part_k<<<dim3(cb, (unsigned)nch), 256, 0, st>>>(src, dt, rows, cols, ld, rpc, scratch);
  colsum_fin_k<<<nblocks(cols), 256, 0, st>>>(scratch, (int)nch, cols, out);
  g_launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ softmax
__global__ void softmax_rows_k(const float* S, void* P, int dt, int64_t rows, int n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* s = S + r * n;
    float mx = -INFINITY;
    for (int c = lane; c < n; c += 32) mx = fmaxf(mx, s[c]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int c = lane; c < n; c += 32) sum += __expf(s[c] - mx);
    const float inv = 1.f / warp_sum(sum);
    for (int c = lane; c < n; c += 32) st_from_f32(P, r * n + c, dt, __expf(s[c] - mx) * inv);
  }
}
cudaError_t softmax_rows(const float* S, void* P, int dt, int64_t rows, int n, cudaStream_t st) {
  softmax_rows_k<<<nblocks(rows, 8, 148 * 64), 256, 0, st>>>(S, P, dt, rows, n);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void softmax_bwd_k(const void* P, const float* dP, void* dS, int dt, int64_t rows, int n, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    float s = 0.f;
    for (int c = lane; c < n; c += 32) s += ld_as_f32(P, r * n + c, dt) * dP[r * n + c];
    s = warp_sum(s);
    for (int c = lane; c < n; c += 32) {
      float p = ld_as_f32(P, r * n + c, dt);
      st_from_f32(dS, r * n + c, dt, scale * p * (dP[r * n + c] - s));
    }
  }
}
cudaError_t softmax_bwd(const void* P, const float* dP, void* dS, int dt, int64_t rows, int n, float scale,
                        cudaStream_t st) {
  softmax_bwd_k<<<nblocks(rows, 8, 148 * 64), 256, 0, st>>>(P, dP, dS, dt, rows, n, scale);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ DCN backward elementwise
__global__ void dcn_bwd_elem_k(const void* dT, const void* X, const void* A, void* dA, float* acc, int dt, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    float g = ld_as_f32(dT, t, dt), x = ld_as_f32(X, t, dt), a = ld_as_f32(A, t, dt);
    st_from_f32(dA, t, dt, g * x);
    acc[t] += g * a + g;
  }
}
cudaError_t dcn_bwd_elem(const void* dT, const void* X, const void* A, void* dA, float* acc, int dt, int64_t n,
                         cudaStream_t st) {
  dcn_bwd_elem_k<<<nblocks(n), 256, 0, st>>>(dT, X, A, dA, acc, dt, n);
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
  conv_fwd_k<<<nblocks((int64_t)B * m * d), 256, 0, st>>>(X, K, pdt, C, k, B, m, d, T, dt);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void conv_dgrad_k(const void* dT, const void* K, int pdt, int C, int k, int B, int m, int d, float* acc,
                             int dt) {
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
  conv_dgrad_k<<<nblocks((int64_t)B * m * d), 256, 0, st>>>(dT, K, pdt, C, k, B, m, d, acc, dt);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void conv_wgrad_k(const void* dT, const void* X, int k, int B, int m, int d, int dt, float* part,
                             int64_t per_block) {
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
  int64_t total = (int64_t)B * m * d;
  int nb = (int)std::min<int64_t>(std::max<int64_t>(1, total / 4096), 148 * 4);
  nb = (int)std::min<int64_t>(nb, (int64_t)(scratch_bytes / (sizeof(float) * k * k)));
  int64_t per = (total + nb - 1) / nb;
  nb = (int)((total + per - 1) / per);
  conv_wgrad_k<<<nb, 256, 0, st>>>(dT, X, k, B, m, d, dt, scratch, per);
  conv_wgrad_fin_k<<<1, 64, 0, st>>>(scratch, nb, C, k * k, dK);
  g_launches += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ head + loss
__global__ void head_k(const void* Y, const void* w, const void* bh, int pdt, const float* labels, int m, int d, int Bg,
                       void* dY, int dt, float* pooled, float* z, float* lossb, float* dz, int do_bwd) {
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
  const int b0 = blockIdx.x * per, b1 = min(B, b0 + per);
  for (int c = threadIdx.x; c < d + 2; c += blockDim.x) {
    float s = 0.f;
    for (int b = b0; b < b1; ++b) {
      s += c < d ? dz[b] * pooled[(int64_t)b * d + c] : (c == d ? dz[b] : lossb[b]);
    }
    part[(int64_t)blockIdx.x * (d + 2) + c] = s;
  }
}
__global__ void head_fin_k(const float* part, int nparts, int d, int Bg, float* loss_out, float* dw, float* db) {
  for (int c = threadIdx.x; c < d + 2; c += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < nparts; ++q) s += part[(int64_t)q * (d + 2) + c];
    if (c < d) dw[c] += s;
    else if (c == d) db[0] += s;
    else if (loss_out) *loss_out = s / (float)Bg;
  }
}
cudaError_t head_fwd_bwd(const void* Y, const void* w, const void* bh, int pdt, const float* labels, int B, int m, int d,
                         int Bg, void* dY, int dt, float* pooled, float* z, float* lossb, float* dz, float* loss_out,
                         float* dw, float* db, int do_bwd, cudaStream_t st) {
  head_k<<<B, 256, 0, st>>>(Y, w, bh, pdt, labels, m, d, Bg, dY, dt, pooled, z, lossb, dz, do_bwd);
  ++g_launches;
  if (do_bwd) {
    const int per = 32, nparts = (B + per - 1) / per;
    float* part = pooled + (int64_t)B * d;   // scratch after pooled (sized by the runtime)
    head_part_k<<<nparts, 128, 0, st>>>(pooled, dz, lossb, B, d, per, part);
    head_fin_k<<<1, 256, 0, st>>>(part, nparts, d, Bg, loss_out, dw, db);
    g_launches += 2;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ SGD, casts, init
__global__ void sgd_cast_k(float* master, const float* grad, float lr, void* copy, int dt, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    float v = master[t];
    if (grad) { v -= lr * grad[t]; master[t] = v; }
    if (copy) st_from_f32(copy, t, dt, v);
  }
}
cudaError_t sgd_cast(float* master, const float* grad, float lr, void* copy, int dt, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  sgd_cast_k<<<nblocks(n), 256, 0, st>>>(master, grad, lr, copy, dt, n);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void cast_k(const void* src, int sdt, void* dst, int ddt, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    st_from_f32(dst, t, ddt, ld_as_f32(src, t, sdt));
}
cudaError_t cast(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cast_k<<<nblocks(n), 256, 0, st>>>(src, sdt, dst, ddt, n);
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
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = splitmix64(seed ^ splitmix64(sid * 0x100000001B3ull + (unsigned long long)(idx0 + t)));
    float u = (float)((h >> 40) * (1.0 / 16777216.0));   // [0,1)
    p[t] = bound * (2.f * u - 1.f);
  }
}
cudaError_t init_uniform(float* p, int64_t n, float bound, unsigned long long seed, unsigned long long stream_id,
                         int64_t idx0, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  init_uniform_k<<<nblocks(n), 256, 0, st>>>(p, n, bound, seed, stream_id, idx0);
  ++g_launches;
  return cudaGetLastError();
}
__global__ void fill_k(float* p, int64_t n, float v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) p[t] = v;
}
cudaError_t fill(float* p, int64_t n, float v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fill_k<<<nblocks(n), 256, 0, st>>>(p, n, v);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace dhen
