// gemm_dispatch.cu — routes each contraction to the tcgen05/TMA kernel when its
// dtype, layouts and alignment allow, else to the exact SIMT kernel.
// DHEN_GEMM=simt forces the SIMT path (A/B measurements only).
#include <cstdlib>
#include <cstring>

#include "gemm.h"

namespace dhen {

int g_last_gemm_tc = 0;
int g_last_gemm_grid = 0;
int pdl_enabled() {
  static int v = [] { const char* e = getenv("DHEN_PDL"); return e ? atoi(e) : 0; }();
  return v;
}
int g_gemm_force = -1;   // -1: env / auto, 0: auto, 1: SIMT only, 2: tcgen05 only
int g_gemm_pair = -1;    // -1: env DHEN_PAIR / auto, 0: no CTA pairs, 1: CTA pairs wherever expressible

static int force_mode() {
  if (g_gemm_force >= 0) return g_gemm_force;
  const char* e = getenv("DHEN_GEMM");
  return (e && !strcmp(e, "simt")) ? 1 : 0;
}

cudaError_t gemm_run(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  g_last_gemm_tc = 0;
  const int mode = force_mode();
  if (mode != 1) {
    cudaError_t e = gemm_tc(g, ws, st);
    if (e == cudaSuccess) { g_last_gemm_tc = g_last_gemm_pair ? 2 : 1; return e; }
    if (e != cudaErrorNotSupported || mode == 2) return e;
  }
  return gemm_simt(g, ws, st);
}

}  // namespace dhen
