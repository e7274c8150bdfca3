// gemm_epi.cuh — the fused GEMM epilogue shared by the SIMT and tcgen05 paths:
// out = alpha*acc (+bias[j]) [aux <- out; out = x*out + x] (relu) (*mask>0) (+resid) (+C).
#pragma once
#include "gemm.h"

namespace dhen {

static __device__ __forceinline__ void epi_apply(const Gemm& g, int z, int i, int j, float acc) {
  const Epilogue& e = g.e;
  if (e.triu_m) {
    const int64_t zb = (int64_t)z * g.c.bs0;
    if (j <= i) return;
    const int64_t o = zb + (int64_t)i * e.triu_m - (int64_t)i * (i + 1) / 2 + (j - i - 1);
    st_from_f32(g.c.ptr, o, g.c.dt, acc * e.alpha);
    return;
  }
  if (e.dcn_bwd) {
    const float v = acc * e.alpha;
    const float x = ld_as_f32(e.cross.ptr, e.cross.off(z, i, j), e.cross.dt);
    const float a = ld_as_f32(e.mask.ptr, e.mask.off(z, i, j), e.mask.dt);
    st_from_f32(e.aux.ptr, e.aux.off(z, i, j), e.aux.dt, v * x);
    const int64_t co = g.c.off(z, i, j);
    const float base = e.resid.ptr ? ld_as_f32(e.resid.ptr, e.resid.off(z, i, j), e.resid.dt)   // first writer
                                   : ld_as_f32(g.c.ptr, co, g.c.dt);
    st_from_f32(g.c.ptr, co, g.c.dt, base + v * a + v);
    return;
  }
  float v = acc * e.alpha;
  if (e.bias) {
    int bj = j;
    bool has = true;
    if (e.bias_gap_hi > e.bias_gap_lo) {
      if (j >= e.bias_gap_lo && j < e.bias_gap_hi) has = false;
      else if (j >= e.bias_gap_hi) bj = j - e.bias_gap_hi + e.bias_hi_off;
    }
    if (has) v += ld_as_f32(e.bias, bj, e.bias_dt);
  }
  if (e.cross.ptr) {
    if (e.aux.ptr) st_from_f32(e.aux.ptr, e.aux.off(z, i, j), e.aux.dt, v);
    float x = ld_as_f32(e.cross.ptr, e.cross.off(z, i, j), e.cross.dt);
    v = x * v + x;
  } else if (e.aux.ptr) {
    st_from_f32(e.aux.ptr, e.aux.off(z, i, j), e.aux.dt, v);
  }
  if (e.relu) v = fmaxf(v, 0.f);
  if (e.mask.ptr) {
    float mv = ld_as_f32(e.mask.ptr, e.mask.off(z, i, j), e.mask.dt);
    v = mv > 0.f ? v : 0.f;
  }
  if (e.resid.ptr) v += ld_as_f32(e.resid.ptr, e.resid.off(z, i, j), e.resid.dt);
  int64_t co = g.c.off(z, i, j);
  if (e.accumulate) v += ld_as_f32(g.c.ptr, co, g.c.dt);
  st_from_f32(g.c.ptr, co, g.c.dt, v);
}

}  // namespace dhen
