// gemm.h — the generic strided/batched contraction every DHEN step lowers to.
//
//   C[z][i][j]  (epilogue)=  alpha * sum_k A[z][i][k] * B[z][k][j]
//
// A, B are bf16 or fp32 (same dtype); accumulation is fp32 (TMEM on the
// tcgen05 path, registers on the SIMT path; never TF32).  Each operand is a
// strided view; the K index may be two-level (k -> (k / kdiv, k % kdiv)) so a
// reduction over (sample, dim) pairs — the token-mixing weight gradients,
// B4/B3 in SURVEY §8(a) — is one GEMM.  The epilogue fuses bias (with an
// optional zero gap, for the key-bias-free QKV projection, R10), the DCN cross
// x ⊙ (acc + b) + x (F8), ReLU, ReLU-mask (backward), residual add and
// accumulation (+=) into C.
#pragma once
#include "common.cuh"

namespace dhen {

struct Operand {            // A: (z, i, k) ; B: (z, k, j)
  const void* ptr;
  int dt;
  int64_t s_mn;             // stride of i (A) / j (B)  (inner index when mdiv > 0)
  int64_t s_k;              // stride of the inner k index
  int64_t s_ko;             // stride of the outer k index (k / kdiv); kdiv == 0: single-level
  int kdiv;
  int64_t bs0, bs1;         // batch strides (z / zdiv, z % zdiv)
  int zdiv;
  int mdiv;                 // two-level i / j: (i / mdiv) * s_mo + (i % mdiv) * s_mn; 0: single-level
  int64_t s_mo;
  __host__ __device__ int64_t off(int64_t z, int64_t mn, int64_t k) const {
    int64_t ko = kdiv ? (k / kdiv) : 0, ki = kdiv ? (k % kdiv) : k;
    int64_t o = ki * s_k + ko * s_ko;
    if (zdiv == 1) o += z * bs0; else o += (z / zdiv) * bs0 + (z % zdiv) * bs1;
    if (mdiv) o += (mn / mdiv) * s_mo + (mn % mdiv) * s_mn; else o += mn * s_mn;
    return o;
  }
};

inline Operand operand(const void* p, int dt, int64_t s_mn, int64_t s_k, int64_t bs0 = 0, int64_t bs1 = 0,
                       int zdiv = 1, int kdiv = 0, int64_t s_ko = 0) {
  Operand o;
  o.ptr = p; o.dt = dt; o.s_mn = s_mn; o.s_k = s_k; o.s_ko = s_ko; o.kdiv = kdiv;
  o.bs0 = bs0; o.bs1 = bs1; o.zdiv = zdiv;
  o.mdiv = 0; o.s_mo = 0;
  return o;
}
// operand with a two-level row index (i -> (i / mdiv, i % mdiv))
inline Operand operand2(const void* p, int dt, int mdiv, int64_t s_mo, int64_t s_mn, int64_t s_k) {
  Operand o = operand(p, dt, s_mn, s_k);
  o.mdiv = mdiv; o.s_mo = s_mo;
  return o;
}

struct Epilogue {
  float alpha = 1.f;
  const void* bias = nullptr;   // indexed by j, dtype bias_dt
  int bias_dt = F32;
  int bias_gap_lo = 0, bias_gap_hi = 0;   // j in [lo, hi) -> no bias; j >= hi -> bias[j - hi + bias_hi_off]
  int bias_hi_off = 0;                    // where column hi's bias lives (relative to bias)
  int relu = 0;
  View mask = noview();         // out *= (mask > 0)           (ReLU backward)
  View cross = noview();        // DCN: aux <- out; out = x * out + x
  View aux = noview();
  View resid = noview();        // out += resid
  int accumulate = 0;           // out += C (C read in its own dtype)
  // DCN backward fused into the token-mixing dgrad (B8): v = acc (= dT); aux <- v * x (dA, x = cross view);
  // C += v * a + v (a = mask view holds A; C is the fp32 dX accumulator)
  int dcn_bwd = 0;
  // with dcn_bwd (tcgen05 path, N <= 256): column sums of dA, one fixed-order partial row per CTA into
  // bsum[blockIdx][N] (the bias gradient's partials; g_last_gemm_grid rows are written)
  float* bsum = nullptr;
  // bf16 C on the TMA-store path: column sums of the STORED C over each 32-row block, written to
  // csum[(z * ceil(M / 32) + row / 32) * N + col] (a bias gradient's partial rows)
  float* csum = nullptr;
  // Gram triangle (F1): element (i, j) of sample z is stored iff j > i, at C + z * c.bs0 +
  // i * triu_m - i (i + 1) / 2 + (j - i - 1)  (strict upper triangle, row-major pairs, R7)
  int triu_m = 0;
  // LayerNorm over the output row (F5 / F6 / F12 fused, N = the whole row): v = alpha acc + bias + resid;
  // aux <- v (bf16, the saved pre-norm sum); C = gamma (v - mu) rstd + beta; mu / rstd (fp32 per row) saved
  const void* ln_gamma = nullptr;
  const void* ln_beta = nullptr;
  float* ln_mu = nullptr;
  float* ln_rstd = nullptr;
  float ln_eps = 1e-5f;
  int ln_d = 0;   // segment (token) length: N (one token per row) or a divisor of N (several tokens per row)
  // ReLU bitmask, word-major [N / 32][bits_ld >= M] (bit j of word (w, r) = column 32 w + j of row r; a warp's
  // lanes = consecutive rows touch consecutive words): bits_mode 1 writes (stored value > 0)
  // next to C (the FFN1 forward), 2 multiplies by it (the FFN2 data gradient) instead of reading the bf16 mask
  uint32_t* bits = nullptr;
  int bits_mode = 0;
  int64_t bits_ld = 0;
};

struct Gemm {
  int M, N, K, batch;
  Operand a, b;
  View c;
  Epilogue e;
};

struct Workspace {              // scratch for split-K partials (fp32)
  float* ptr = nullptr;
  size_t bytes = 0;
};

// Launch counter (reported as gpu_launches by the bench).
extern unsigned long long g_launches;
// 1 if the last gemm_run took the tcgen05 path (profiling attribution).
extern int g_last_gemm_tc;
extern int g_last_gemm_grid;   // CTAs of the last tcgen05 GEMM launch (rows of an Epilogue::bsum partial)
extern thread_local int g_gemm_pair;
extern int g_last_gemm_pair;
// path override of dhen_debug_gemm: -1 the switches, 0 auto, 1 SIMT only, 2 tcgen05 only
extern thread_local int g_gemm_force;
// debug: device buffer of >= 448 int64 for a clock64 trace of CTA 0 of the next tcgen05 GEMMs
extern long long* g_gemm_trace;

// Dispatch: tcgen05/TMA path when the shapes and layouts allow it, the SIMT
// path (exact fp32 FMA; the fp32 mode and odd shapes) otherwise.
cudaError_t gemm_run(const Gemm& g, const Workspace& ws, cudaStream_t st);
cudaError_t gemm_simt(const Gemm& g, const Workspace& ws, cudaStream_t st);
// tcgen05 path; returns cudaErrorNotSupported (nothing launched) when the GEMM does not qualify.
cudaError_t gemm_tc(const Gemm& g, const Workspace& ws, cudaStream_t st);
// sums split-K partials ws[(z*splits+sp)][M][N] in fixed order and applies the epilogue.
cudaError_t splitk_reduce(const Gemm& g, int splits, const float* ws, cudaStream_t st);

}  // namespace dhen
