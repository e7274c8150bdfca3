// dcn_bwd.h — B8 (the DCN cross backward) as one kernel per 128-row tile (dcn_bwd_tc.cu; Eq.(7), R13).
//   Wu: bf16 W_u [m][l] (m = 128) or its block-diagonal form [128][spt l] (m = 128 / spt); dU: bf16 [B][l][d]
//   (sample stride ldu); W: bf16 [d][d]; X, A: bf16 [B m][d]; rin: bf16 dR (first writer) or fp32 accumulator;
//   out: fp32 accumulator or bf16 dX; dA: bf16 [B m][d] out; bsum (nullable): fp32 [rows][d] partial column sums
//   of dA (*rows_out rows, to be added in order).  cudaErrorNotSupported (nothing launched) outside d in
//   {128, 256}, m dividing 128, B a multiple of spt, 16 | K1 = spt l with K1 d 2 <= 16 KB, or K1 <= 128 with a bf16
//   base and bf16 dX (the shared-tile form).
#pragma once
#include "common.cuh"

namespace dhen {
extern unsigned long long g_launches;
namespace dcnb {
bool supported(int B, int m, int l, int d, int64_t ldu, int rin_f32, int out_f32);
cudaError_t bwd(const void* Wu, const void* dU, int64_t ldu, const void* W, const void* X, const void* A, const void* rin,
                int rin_f32, void* out, int out_f32, void* dA, float* bsum, int B, int m, int l, int d, cudaStream_t st,
                int* rows_out);
}  // namespace dcnb
}  // namespace dhen
