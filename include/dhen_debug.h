/* dhen_debug.h — test and debugging hooks of libdhen.so (not part of the training API in dhen.h).
 *
 * These reach below the layer calls: one GEMM through the library's dispatcher (with or without a fused
 * epilogue), a clock64 trace of the tcgen05 GEMM's pipeline, a context's schedule / fusion switches
 * (dhen_tuning) and a per-op timeline dump.  Used by tests/test_gpu_gemm.py, tests/test_gpu_attn.py,
 * tests/test_gpu_fusions.py and tools/; nothing on the training path calls them.
 */
#ifndef DHEN_DEBUG_H_
#define DHEN_DEBUG_H_

#include <stddef.h>

#include "dhen.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Test hook (tests/test_gpu_gemm.py): one strided / batched contraction
 *   C[z][i][j] (+)= sum_k A[z][i][k] B[z][k][j]
 * through the library's GEMM dispatcher.  q = int64[30]: M, N, K, batch,
 * A{s_mn, s_k, bs0, bs1, zdiv, kdiv, s_ko}, B{s_mn, s_k, bs0, bs1, zdiv, kdiv, s_ko},
 * C{rs, cs, bs0, bs1, zdiv}, accumulate, A{mdiv, s_mo}, B{mdiv, s_mo}, C{rdiv, rs_o}
 * (two-level row index r -> (r / div) * s_o + (r % div) * s; div 0 = single level).  ab_dtype/c_dtype: dhen_dtype.
 * path: 0 auto, 1 SIMT only, 2 tcgen05 only (DHEN_E_CONFIG if not expressible), 3 tcgen05 with CTA pairs
 * (cta_group::2, 256-row tiles) wherever the tile width allows, 4 tcgen05 without CTA pairs.
 * ws: fp32 device scratch for split-K partials. */
dhen_status dhen_debug_gemm(const long long* q, const void* A, const void* B, void* C, int ab_dtype, int c_dtype,
                            int path, void* ws, size_t ws_bytes, void* stream);
/* Test hook: as dhen_debug_gemm plus one fused epilogue: mode 1 ReLU-mask by E (> 0), 2 residual
 * + E, 3 DCN cross E (.) (acc + bias) + E with the pre-cross value stored to aux, 4 ReLU; E / aux are bf16
 * with C's geometry; bias (bf16, nullable) is indexed by column. */
dhen_status dhen_debug_gemm_epi(const long long* q, const void* A, const void* B, void* C, int ab_dtype, int c_dtype,
                                int path, void* ws, size_t ws_bytes, int mode, const void* E, const void* bias,
                                void* aux, void* stream);
/* 0: the last GEMM ran on the SIMT path, 1: tcgen05 (one CTA per tile), 2: tcgen05 with CTA pairs. */
int dhen_debug_last_gemm_tc(void);
/* Debug: device buffer (>= 448 int64) receiving clock64 timestamps of CTA 0 of every following
 * tcgen05 GEMM (producer issue, MMA start, data ready, epilogue start, epilogue end); NULL = off. */
void dhen_debug_gemm_trace(void* dev_buf);

/* Schedule / fusion switches of one context (A/B measurements and the fusion tests).  Every field's
 * default (dhen_tuning_default) is the measured-best setting; each alternative computes the same function
 * (bitwise, or within bf16 rounding where a fusion moves a rounding point -- tests/test_gpu_fusions.py).
 * Nothing is read from the environment: a context's switches are its own, so one process can A/B them. */
typedef struct {
  int overlap;       /* 1: module branches / weight gradients on a second stream                      (1) */
  int defer_join;    /* 1: side-stream joins deferred until a shared buffer is reused                 (1) */
  int ln_fuse;       /* 1: LayerNorm (F5, F6, F12) in the producing GEMM epilogues                     (1) */
  int first_writer;  /* 1: the first module's dX GEMM adds dR, the last one emits bf16 dX (B3, B10)    (1) */
  int relu_bits;     /* 1: the FFN ReLU derivative from a bitmask written by FFN1                      (1) */
  int fuse_db;       /* 1: DCN db / FFN db_1 from column sums in GEMM epilogues                        (1) */
  int vdy;           /* 1: the head's dY formed inside the last layer's LayerNorm backward             (1) */
  int trail;         /* 1: LayerNorm / head parameter sums trail on the side stream                    (1) */
  int bd_pre;        /* 1: every layer's block-diagonal token maps built by one launch per step        (1) */
  int sym;           /* Gram-backward symmetrisation: -1 by m (dense image for m >= 128), 0 staged
                        triangle, 1 dense image (triangle staged in smem), 2 dense image from global   (-1) */
  int tstore;        /* 1: TMA-store GEMM epilogue where the epilogue allows it                        (1) */
  int pair;          /* CTA pairs (cta_group::2): -1 size rule, 0 never, 1 wherever expressible      (-1) */
  int pair_k;        /* the size rule's K threshold                                                 (1024) */
  int attn_fused;    /* 1: fused tcgen05 attention core (m <= 128, dh 64 / 128); 0: 2 GEMMs + softmax  (1) */
  int pdl;           /* 1: programmatic dependent launch on every library launch                        (0) */
  int gemm_simt;     /* 1: every GEMM on the exact-fp32 SIMT path (never in bf16 production)           (0) */
  int dcn_fused;     /* 1: DCN backward as one kernel where the shape allows (dT, dA, dA W; the partial dX
                        kept in TMEM, W streamed, operands / outputs as TMA boxes; bit-identical);
                        0: two GEMMs with an fp32 partial dX in HBM.  C5 +20 %, C2 +9 %, C4 +2 %        (1) */
  int dcn_tma;       /* 1: the DCN-backward dT GEMM's epilogue takes X, A, dR through TMA-loaded shared boxes
                        and stores dA, dX by TMA; 0: per-lane global loads (round 1)                    (1) */
  int ln_tma;        /* 1: LayerNorm GEMM epilogues take the residual by TMA and store R, Y by TMA; 0: register
                        prefetch and staged coalesced stores                                            (1) */
  int bn_max;        /* widest GEMM tile N (64 / 128 / 256); smaller tiles trade per-tile efficiency for
                        more tiles (wave quantization of short grids)                                 (256) */
  int l2_prefetch;   /* short-K GEMMs (K <= 512): the TMA producer prefetches the operand tiles of the CTA's
                        item this many items ahead into L2 (cp.async.bulk.prefetch.tensor); 0 off, <= 4 */
  int wres;          /* short-K TMA-store GEMMs (K <= 256, BN = 256, bf16 C) keep the weight tile resident in shared
                        memory and stream only A (a third of the L2 reads): 1 one CTA a tile, 2 CTA pairs (each
                        CTA half the tile, an A ring twice as deep), 0 off                              (1) */
  int resid_tma;     /* 1: the fp32-residual GEMM epilogue (token-map dgrad first writer) takes dR through TMA
                        boxes and stores C by TMA; 0: register prefetch and staged stores               (1) */
} dhen_tuning;

void dhen_tuning_default(dhen_tuning* t);
/* Replace ctx's switches (drops a captured step graph).  DHEN_E_CONFIG on an out-of-range field. */
dhen_status dhen_set_tuning(dhen_ctx* ctx, const dhen_tuning* t);
dhen_status dhen_get_tuning(const dhen_ctx* ctx, dhen_tuning* t);

/* Per-op timeline of the last profiled pass (dhen_profile): one CSV line per recorded op
 * (tag, stream index, start ms, end ms relative to the first record) -> path.  tools/timeline.py reads it. */
dhen_status dhen_debug_profile_trace(dhen_ctx* ctx, const char* path);

#ifdef __cplusplus
}
#endif
#endif /* DHEN_DEBUG_H_ */
