// kernels.h — launchers of the non-GEMM DHEN kernels (sm_100a).  Every launcher
// enqueues on `st`, counts its launches in g_launches and returns the launch error.
#pragma once
#include "common.cuh"

namespace dhen {

extern unsigned long long g_launches;

// F1: Z[b][p] = G[b][i][j] for i < j, p row-major (R7).  G fp32 [B][m][m].
cudaError_t triu_extract(const float* G, void* Z, int dt, int B, int m, int64_t ldz, cudaStream_t st);
// B5: S[b][i][j] = S[b][j][i] = dZ[b][p(i,j)], S[b][i][i] = 0.
cudaError_t sym_from_triu(const void* dZ, void* S, int dt, int B, int m, int64_t ldz, cudaStream_t st);

// F12 / encoder LN1, LN2: R = U (+ addx), Y = gamma (R - mu) rstd + beta per row of d.
// U fp32 [rows][d]; addx (dt) nullable; Y, Rsave dtype dt; mu, rstd fp32 [rows].
cudaError_t ln_fwd(const float* U, const void* addx, const void* gamma, const void* beta, int pdt, float eps,
                   int64_t rows, int d, void* Y, void* Rsave, float* mu, float* rstd, int dt, cudaStream_t st);
// B2: dR = rstd (g - mean g - xh mean(g xh)), g = dY * gamma, xh from Rsave.  dR stored (dt);
// acc_mode 1: acc = dR, 2: acc += dR (fp32 rows x d).  dgamma/dbeta += sums (deterministic).
cudaError_t ln_bwd(const void* dY, int dydt, const void* Rsave, const float* mu, const float* rstd,
                   const void* gamma, int pdt, int64_t rows, int d, void* dR, int dt, float* acc, int acc_mode,
                   float* dgamma, float* dbeta, float* scratch, size_t scratch_bytes, cudaStream_t st,
                   cudaStream_t st_red = nullptr, cudaEvent_t ev_red = nullptr, const float* vdz = nullptr,
                   const void* vw = nullptr, int vm = 0);
// (vdz: dY is not read; row r of dY is bf16(vdz[r / vm] / vm * vw) -- the head's gradient, formed in place)
// (st_red: the final fixed-order reduction of the dgamma / dbeta partials runs there, after ev_red is
//  recorded on st; scratch must then stay untouched on st until st_red is joined back)

// out[c] += sum_p part[p * n + c] over p < nparts, in index order (partial rows -> a gradient)
cudaError_t rows_sum_add(const float* part, int nparts, int n, float* out, cudaStream_t st);
// out[c] += sum_r src[r * ld + c] for c < cols (deterministic two-pass).
cudaError_t colsum_add(const void* src, int dt, int64_t rows, int cols, int64_t ld, float* out,
                       float* scratch, size_t scratch_bytes, cudaStream_t st);

// F4 softmax over rows (n valid columns, row pitch ld) of S (fp32) -> P (dt).
// B6: dS = scale * P (dP - rowsum(P dP)).
cudaError_t softmax_rows(const float* S, void* P, int dt, int64_t rows, int n, int ld, cudaStream_t st);
cudaError_t softmax_bwd(const void* P, const float* dP, void* dS, int dt, int64_t rows, int n, int ld, float scale,
                        cudaStream_t st);

// B8 elementwise: dA = dT * X (dt); acc += dT * A + dT.
cudaError_t dcn_bwd_elem(const void* dT, const void* X, const void* A, void* dA, float* acc, int dt, int64_t n,
                         cudaStream_t st);

// F7 / B7: 1-channel m x d image, C k x k filters folded to their mean (exact), zero padding.
cudaError_t conv_fwd(const void* X, const void* K, int pdt, int C, int k, int B, int m, int d, void* T, int dt,
                     cudaStream_t st);
cudaError_t conv_dgrad(const void* dT, const void* K, int pdt, int C, int k, int B, int m, int d, float* acc, int dt,
                       cudaStream_t st);
cudaError_t conv_wgrad(const void* dT, const void* X, int C, int k, int B, int m, int d, int dt, float* dK,
                       float* scratch, size_t scratch_bytes, cudaStream_t st);

// F13 / B1: z_b = w . mean_t Y[b,t] + b_h; loss_b = BCE(z_b, y_b); dz_b = (sigma(z_b) - y_b) / Bg;
// dY[b,t,c] = dz_b w[c] / m (dt).  Then loss_out = sum_b loss_b / Bg, dw += sum dz pooled, db += sum dz.
cudaError_t head_fwd_bwd(const void* Y, const void* w, const void* bh, int pdt, const float* labels, int B, int m, int d,
                         int Bg, void* dY, int dt, float* pooled, float* z, float* lossb, float* dz, float* loss_out,
                         float* dw, float* db, int do_bwd, cudaStream_t st, cudaStream_t st_red = nullptr,
                         cudaEvent_t ev_red = nullptr);

// Several block-diagonal maps in one launch (a training step builds every layer's up front).
struct BdJob {
  const __nv_bfloat16* W;
  __nv_bfloat16* out;
  int m, l, spt, tr;   // tr = 1: blockdiag_t layout, 0: blockdiag layout
};
struct BdJobs {
  int n;
  BdJob job[32];
};
cudaError_t blockdiag_multi(const BdJobs& jobs, cudaStream_t st);
// out (bf16 [spt m][spt l]) = blockdiag(W, .., W) of the bf16 token map W [m][l] (DCN backward packing)
cudaError_t blockdiag(const void* W, int m, int l, int spt, void* out, cudaStream_t st);
// out (bf16 [spt l][spt m]) = blockdiag(W^T, .., W^T) (packed token projection)
cudaError_t blockdiag_t(const void* W, int m, int l, int spt, void* out, cudaStream_t st);

// SGD (R18): master -= lr * grad; copy = (dt) master.  lr == 0 with grad == NULL: refresh copy only.
cudaError_t sgd_cast(float* master, const float* grad, float lr, void* copy, int dt, int64_t n, cudaStream_t st);
cudaError_t cast(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t st);
// multi-tensor SGD (bf16 compute copies): segment s = n4[s] float4 groups of master / grad / copy (<= 32 segments)
struct SgdSegs {
  int n;
  float* master[32];
  const float* grad[32];
  void* copy[32];
  int64_t n4[32];
};
cudaError_t sgd_multi(const SgdSegs& segs, float lr, cudaStream_t st);
// Adam (Kingma & Ba; PyTorch torch.optim.Adam semantics, no weight decay) on an fp32 master shard with fp32
// moments m, v; the step number t is read from *step (device; the update of step t uses t = *step + 1) and
// the compute copy (dt) refreshed.  adam_count(step) increments *step afterwards (graph-replay safe).
cudaError_t adam_step(float* master, const float* grad, void* m, void* v, int mdt, void* copy, int dt, int64_t n, float lr,
                      float b1, float b2, float eps, const int* step, cudaStream_t st);
cudaError_t adam_count(int* step, cudaStream_t st);
// Sum / weighted-sum ensemble (R27).  ens_ln_fwd: R = sum_i w_i U_i + base (w nullable = all 1; base = the
// fp32 W_n projection `base32`, or the identity shortcut `basex` in dt), then the layer LayerNorm (two-pass
// statistics) -> Y (dt), R (dt, saved), mu, rstd.  U: k fp32 [rows][d] buffers.
struct EnsU { const float* u[16]; int k; };
cudaError_t ens_ln_fwd(const EnsU& U, const void* w, int pdt, const float* base32, const void* basex, const void* gamma,
                       const void* beta, float eps, int64_t rows, int d, void* Y, void* R, float* mu, float* rstd, int dt,
                       cudaStream_t st);
// paper-literal DCN backward (R31): S[b][c][k] = dG[b][c][k] + dG[b][k][c] (fp32 in, dt out), d x d per sample
cudaError_t sym_add(const float* dG, void* S, int dt, int B, int d, cudaStream_t st);
// out (dt) = w[i] (pdt) * dR (dt), n elements
cudaError_t ens_scale(const void* dR, const void* w, int i, int pdt, void* out, int64_t n, int dt, cudaStream_t st);
// *acc += sum_j U[j] dR[j] (fixed-order two-pass reduction through `scratch` >= 4 KB)
cudaError_t ens_dot(const float* U, const void* dR, int dt, int64_t n, float* acc, float* scratch, cudaStream_t st);
// parameter init: uniform(-bound, bound) from a counter-based hash of (seed, index), or a constant.
// element i gets the value of tensor index idx0 + i (sharded init gives the same tensor at any world size)
cudaError_t init_uniform(float* p, int64_t n, float bound, unsigned long long seed, unsigned long long stream_id,
                         int64_t idx0, cudaStream_t st);
cudaError_t fill(float* p, int64_t n, float v, cudaStream_t st);
// Dense-token injection (R38): Xin[b] = [X[b] (mi rows) ; X0[b][0 .. nD)]; backward: dD[b] += accm[b][mi ..];
// dX[b][t] = dt(acc_sc[b][t] + accm[b][t] (+ dD[b][t] for t < nDadd)), accm rows of pitch m_mod.
cudaError_t inject_copy(const void* X, const void* X0, int dt, int64_t B, int mi, int nD, int m0, int d, void* Xin,
                        cudaStream_t st);
cudaError_t inject_dD(const float* accm, int64_t B, int mi, int nD, int d, float* dD, cudaStream_t st);
cudaError_t inject_final(const float* acc_sc, const float* accm, int m_mod, const float* dD, int nDadd, int64_t B, int mi,
                         int d, void* dX, int dt, cudaStream_t st);

}  // namespace dhen
