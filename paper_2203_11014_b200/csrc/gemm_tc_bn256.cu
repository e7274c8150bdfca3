// gemm_tc_bn256.cu — instantiations of the tcgen05 GEMM kernel for BN = 256 (all epilogue variants).
#include "gemm_tc_kernel.cuh"

namespace dhen {
namespace tc {
cudaError_t launch_bn256(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, const OutMaps& mc,
                        cudaStream_t st, int var) {
  return launch_var<256, 3>(p, ma, mb, mc, st, var);
}
}  // namespace tc
}  // namespace dhen
