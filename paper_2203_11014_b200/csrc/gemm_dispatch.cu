// gemm_dispatch.cu — routes each contraction to the tcgen05/TMA kernel when its
// dtype, layouts and alignment allow, else to the exact SIMT kernel; and the thread's current
// schedule switches (tuning.h).
#include <cstdlib>
#include <cstring>

#include "gemm.h"
#include "tuning.h"

namespace dhen {

dhen_tuning tuning_default() {
  dhen_tuning t;
  t.overlap = 1; t.defer_join = 1; t.ln_fuse = 1; t.first_writer = 1; t.relu_bits = 1; t.fuse_db = 1; t.vdy = 1;
  t.trail = 1; t.bd_pre = 1; t.sym = -1; t.tstore = 1; t.pair = -1; t.pair_k = 1024; t.attn_fused = 1; t.pdl = 0;
  t.gemm_simt = 0; t.dcn_fused = 1; t.dcn_tma = 1; t.ln_tma = 1; t.bn_max = 256; t.l2_prefetch = 0; t.wres = 1; t.resid_tma = 1;
  return t;
}
static thread_local const dhen_tuning* t_tune = nullptr;
const dhen_tuning& tune() {
  static const dhen_tuning d = tuning_default();
  return t_tune ? *t_tune : d;
}
TuneScope::TuneScope(const dhen_tuning* t) : prev(t_tune) { t_tune = t; }
TuneScope::~TuneScope() { t_tune = prev; }

int g_last_gemm_tc = 0;
int g_last_gemm_grid = 0;
int pdl_enabled() { return tune().pdl; }
thread_local int g_gemm_force = -1;   // dhen_debug_gemm's path: -1 switches, 0 auto, 1 SIMT only, 2 tcgen05 only
thread_local int g_gemm_pair = -1;    // dhen_debug_gemm's path: -1 switches, 0 no CTA pairs, 1 pairs wherever possible

static int force_mode() {
  if (g_gemm_force >= 0) return g_gemm_force;
  return tune().gemm_simt ? 1 : 0;
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
