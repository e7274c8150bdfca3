// attn.h — fused self-attention core (F4 forward, B6 core backward) for m <= 128 tokens, dh in {64, 128}.
// QKV: bf16 [B][m][3d] (Q | K | V, head h at columns h*dh of each third, no padding); O: bf16 [B][m][d];
// dO: bf16 [B][m][d]; dQKV: bf16 [B][m][3d].  Returns cudaErrorNotSupported (nothing launched) when the
// shape is not covered or the context's switches turn it off (dhen_tuning.attn_fused); the caller then takes
// the two-GEMM + softmax path.
#pragma once
#include "common.cuh"

namespace dhen {
extern unsigned long long g_launches;
namespace attn {
bool fused_ok(int dt, int B, int H, int m, int d);
cudaError_t core_fwd(const void* QKV, void* O, int B, int H, int m, int d, cudaStream_t st);
cudaError_t core_bwd(const void* QKV, const void* dO, void* dQKV, int B, int H, int m, int d, cudaStream_t st);
}  // namespace attn
}  // namespace dhen
