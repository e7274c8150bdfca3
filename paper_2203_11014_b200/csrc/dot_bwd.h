// dot_bwd.h — the Gram backward of the Dot module with S built on chip (dot_bwd_tc.cu; B5, Eq.(3)).
//   dZ: bf16 [B][ldz] packed strict upper triangles (ldz == m (m - 1) / 2);  X: bf16 [B m][d] row-major
//   mode 0: out (fp32 [B m][d]) += S X;      mode 1: out (fp32) = rin (bf16 dR) + S X
//   mode 2: out (bf16) = rin (fp32 acc) + S X;  mode 3: out (bf16) = rin (bf16 dR) + S X
// Returns cudaErrorNotSupported (nothing launched) outside d in {128, 256}, m <= 128 with 32 | (samples per
// tile) m, B a multiple of the samples per tile; the caller then takes the dense-S path.
#pragma once
#include "common.cuh"

namespace dhen {
extern unsigned long long g_launches;
namespace dotb {
bool supported(int B, int m, int d, int64_t ldz);
int samples_per_item(int m);
cudaError_t gram_bwd(const void* dZ, int64_t ldz, const void* X, int B, int m, int d, int mode, const void* rin, void* out,
                     cudaStream_t st);
}  // namespace dotb
}  // namespace dhen
