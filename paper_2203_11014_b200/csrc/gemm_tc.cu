// gemm_tc.cu — bf16 GEMM on the 5th-generation tensor cores (sm_100a):
// TMA (cp.async.bulk.tensor, 128B swizzle) fills a multi-stage shared-memory
// ring guarded by mbarriers; one elected thread issues tcgen05.mma
// (kind::f16, M = 128, N = BN, K = 16 per instruction) accumulating in TMEM;
// tcgen05.commit releases ring slots and finally signals the epilogue; four
// warps read the fp32 accumulator back with tcgen05.ld and apply the fused
// epilogue (bias / DCN cross / ReLU / mask / residual / +=).
//
// Operands may be K-major or MN-major (transposed views of row-major tensors,
// so dgrad / wgrad need no transpose kernels), batched through up to two
// batch strides, and may have a two-level K (k -> (k / kdiv, k % kdiv)) so the
// token-mixing weight gradients reduce over (sample, dim) in one GEMM.  Long K
// with few output tiles is split across CTAs with a deterministic fixed-order
// second pass.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gemm_tc_kernel.cuh"
#include "tuning.h"

namespace dhen {
long long* g_gemm_trace = nullptr;
int g_last_gemm_pair = 0;
namespace tc {

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)f;
  }
  return fn;
}

// Build the TMA map of one operand (rows = M for A, N for B).  Returns false if
// the layout is not TMA-expressible (the GEMM then runs on the SIMT path).
static bool make_map(CUtensorMap* map, OpMap* om, const Operand& o, int rows, int K, int batch, int tile_rows) {
  const int64_t es = 2;
  const bool kmaj = (o.s_k == 1), mnmaj = (o.s_mn == 1);
  if (!kmaj && !mnmaj) return false;
  if (((uintptr_t)o.ptr & 15) != 0) return false;
  om->mn_major = kmaj ? 0 : 1;
  om->has_ko = o.kdiv ? 1 : 0;
  om->kdiv = o.kdiv ? o.kdiv : 1;
  om->zdiv = o.zdiv;
  om->z0 = om->z1 = om->mo = -1;
  om->mdiv = o.mdiv ? o.mdiv : 1;
  // two-level K: kdiv a multiple of BK (a k-block inside one outer index), or, MN-major only, kdiv dividing BK
  // (the box spans BK / kdiv outer indices: k-rows land in smem in (outer, inner) = k order)
  const bool ko_in_box = o.kdiv && o.kdiv < BK && BK % o.kdiv == 0 && mnmaj && !kmaj;
  if (o.kdiv && ((o.kdiv % BK != 0 && !ko_in_box) || K % o.kdiv != 0)) return false;
  if (o.mdiv && (o.mdiv % tile_rows != 0 || rows % o.mdiv != 0)) return false;
  cuuint64_t dims[5] = {1, 1, 1, 1, 1}, strides[4] = {0, 0, 0, 0};
  cuuint32_t box[5] = {1, 1, 1, 1, 1}, estr[5] = {1, 1, 1, 1, 1};
  const int kin = o.kdiv ? o.kdiv : K;
  int64_t s1;
  const int rin = o.mdiv ? o.mdiv : rows;
  if (!om->mn_major) {
    dims[0] = kin; dims[1] = rin; s1 = o.s_mn;
    box[0] = BK; box[1] = tile_rows;
  } else {
    dims[0] = rin; dims[1] = kin; s1 = o.s_k;
    box[0] = 64; box[1] = BK;
  }
  strides[0] = s1 * es;
  int r = 2;
  if (o.kdiv) {
    dims[r] = K / o.kdiv; strides[r - 1] = o.s_ko * es;
    if (ko_in_box) { box[1] = o.kdiv; box[r] = BK / o.kdiv; }
    ++r;
  }
  if (o.mdiv) { dims[r] = rows / o.mdiv; strides[r - 1] = o.s_mo * es; om->mo = r; ++r; }
  if (o.zdiv > 1 && o.bs1 != 0) { dims[r] = o.zdiv; strides[r - 1] = o.bs1 * es; om->z1 = r; ++r; }
  const int nb0 = (batch + o.zdiv - 1) / o.zdiv;
  if (nb0 > 1 && o.bs0 != 0) {
    if (r >= 5) return false;
    dims[r] = nb0; strides[r - 1] = o.bs0 * es; om->z0 = r; ++r;
  }
  if (r > 5) return false;
  for (int i = 0; i < 4; ++i) {
    if (i + 1 >= r) strides[i] = (i == 0 ? 16 : strides[i - 1]) ;
    if (strides[i] % 16 != 0 || strides[i] == 0 || strides[i] >= (1ull << 40)) return false;
  }
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  CUresult res = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(o.ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

static bool same_geom(const View& a, const View& c, bool allow_f32 = false) {
  return !a.ptr || (a.rs == c.rs && a.cs == c.cs && a.bs0 == c.bs0 && a.bs1 == c.bs1 && a.zdiv == c.zdiv &&
                    a.rdiv == c.rdiv && a.rs_o == c.rs_o && (a.dt == BF16 || (allow_f32 && a.dt == F32)));
}
// Resolve the epilogue to a Lean plan: all present views share C's geometry, operands other than C
// are bf16, and row-major outputs have N % 4 == 0 with 4-element-aligned rows (vector accesses).
static bool make_lean(const Gemm& g, Lean* e) {
  const Epilogue& x = g.e;
  // an fp32 residual is the dX accumulator read by its last writer (bf16 C, no other fused operand)
  const bool r32 = x.resid.ptr && x.resid.dt == F32;
  if (r32 && (g.c.dt != BF16 || x.cross.ptr || x.mask.ptr || x.aux.ptr || x.bias || x.accumulate || x.relu ||
              x.dcn_bwd || x.triu_m || x.ln_gamma || x.bits_mode))
    return false;
  if (!same_geom(x.cross, g.c) || !same_geom(x.aux, g.c) || !same_geom(x.mask, g.c) || !same_geom(x.resid, g.c, r32))
    return false;
  if (x.bias && x.bias_dt != BF16) return false;
  if (g.c.cs == 1 && !x.triu_m && (g.N % 4 || g.c.rs % 4 || g.c.bs0 % 4 || g.c.bs1 % 4 || g.c.rs_o % 4)) return false;
  auto al = [](const void* p, int b) { return !p || ((uintptr_t)p % b) == 0; };
  if (g.c.cs == 1 && !x.triu_m && (!al(g.c.ptr, g.c.dt == F32 ? 16 : 8) || !al(x.cross.ptr, 8) || !al(x.aux.ptr, 8) ||
                      !al(x.mask.ptr, 8) || !al(x.resid.ptr, 8)))
    return false;
  e->c = g.c.ptr; e->x = x.cross.ptr; e->aux = x.aux.ptr; e->mask = x.mask.ptr; e->resid = x.resid.ptr;
  e->bias = x.bias;
  e->rs = g.c.rs; e->rs_o = g.c.rs_o; e->bs0 = g.c.bs0; e->bs1 = g.c.bs1; e->cs = g.c.cs;
  e->rdiv = g.c.rdiv; e->zdiv = g.c.zdiv;
  e->c_f32 = g.c.dt == F32;
  e->alpha = x.alpha;
  e->gap_lo = x.bias_gap_lo; e->gap_hi = x.bias_gap_hi; e->hi_off = x.bias_hi_off;
  e->flags = (x.accumulate ? EF_ACC : 0) | (x.relu ? EF_RELU : 0) | (x.mask.ptr ? EF_MASK : 0) |
             (x.cross.ptr ? EF_CROSS : 0) | (x.aux.ptr ? EF_AUX : 0) | (x.resid.ptr ? EF_RESID : 0) |
             (x.bias ? EF_BIAS : 0) | (r32 ? EF_R32 : 0);
  e->ln_gamma = x.ln_gamma; e->ln_beta = x.ln_beta; e->ln_mu = x.ln_mu; e->ln_rstd = x.ln_rstd; e->ln_eps = x.ln_eps;
  e->ln_d = x.ln_d ? x.ln_d : g.N;
  e->bits = x.bits; e->bits_ld = x.bits_ld;
  if (x.bits_mode) {
    if (g.c.dt != BF16 || g.N % 64 || g.batch != 1 || x.mask.ptr || (x.bits_mode == 1 && !x.relu)) return false;
    e->flags |= x.bits_mode == 1 ? EF_BITS : EF_BMASK;
  }
  if (x.ln_gamma) {   // LayerNorm epilogue: token segments in one tile, bf16 output, residual, pre-norm sum to aux
    if (g.c.dt != BF16 || g.c.cs != 1 || !x.resid.ptr || !x.aux.ptr || !x.ln_beta || !x.ln_mu || !x.ln_rstd ||
        x.accumulate || x.relu || x.mask.ptr || x.cross.ptr || x.triu_m || x.dcn_bwd)
      return false;
    e->flags |= EF_LN;
  }
  e->triu_m = x.triu_m;
  e->bsum = x.dcn_bwd ? x.bsum : nullptr;
  e->csum = x.csum;
  if (x.dcn_bwd) {
    if (g.c.dt != F32 || !x.cross.ptr || !x.mask.ptr || !x.aux.ptr || x.bias || x.accumulate) return false;
    e->flags = EF_DCNB | (x.resid.ptr ? EF_RESID : 0);   // with a residual: first writer (C = resid + ...)
  }
  if (x.triu_m) {
    if (g.c.rs != 0 || g.c.rdiv || g.c.zdiv != 1 || x.bias || x.accumulate || x.cross.ptr || x.mask.ptr ||
        x.resid.ptr || x.aux.ptr || x.relu)
      return false;
    e->flags = EF_TRIU;
  }
  return true;
}

// a view can take 4-wide vector accesses: column-contiguous rows, every row / batch offset a multiple of 4
// elements and a base aligned to 4 elements of its dtype
static bool vec_ok(const View& v) {
  if (!v.ptr) return true;
  const int es = v.dt == F32 ? 4 : 2;
  if (v.cs != 1) return false;
  if (((uintptr_t)v.ptr) % (4 * es)) return false;
  if (v.rs % 4 || v.bs0 % 4 || v.bs1 % 4 || v.rs_o % 4) return false;
  return true;
}

}  // namespace tc

cudaError_t gemm_tc(const Gemm& g, const Workspace& ws, cudaStream_t st) {
  using namespace tc;
  if (g.a.dt != BF16 || g.b.dt != BF16 || g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return cudaErrorNotSupported;
  if (g.N < 16) return cudaErrorNotSupported;
  const int BN0 = g.N <= 64 ? 64 : g.N <= 128 ? 128 : 256;
  // dhen_tuning.bn_max caps the tile width, except where a LayerNorm segment needs the wider tile
  const int BN = (g.e.ln_gamma && (g.e.ln_d ? g.e.ln_d : g.N) > std::min(tune().bn_max, BN0)) ? BN0
                                                                                            : std::min(tune().bn_max, BN0);
  if (g.e.ln_gamma) {   // LN segments must be whole warp halves or whole tiles, and tiles must be full
    const int ld_ = g.e.ln_d ? g.e.ln_d : g.N;
    if (BN < 128 || g.N % BN != 0 || (ld_ != BN && ld_ != BN / 2)) return cudaErrorNotSupported;
  }
  Params p;
  p.g = g;
  p.tiles_m = (g.M + BM - 1) / BM;
  p.tiles_n = (g.N + BN - 1) / BN;
  p.kblocks = (g.K + BK - 1) / BK;
  const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n * g.batch;
  int splits = 1;
  if (tiles * 2 <= 148 && p.kblocks >= 8 && !g.e.ln_gamma) {   // output fills < half the SMs, long K: split K
    // one item per SM: floor, so tiles x splits never exceeds the SM count (a 149th item doubles the time)
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(148 / tiles, p.kblocks / 4));
    while (splits > 1 && (int64_t)splits * g.batch * g.M * g.N * 4 > (int64_t)ws.bytes) --splits;
  }
  // CTA pairs (cta_group::2, 256 x BN tiles, each CTA loads BN / 2 rows of B): halves the B bytes per ring
  // slot, so the same shared memory holds a deeper ring (BN = 256: 4 slots instead of 3).  Measured
  // (tools/gemm_bench.py, dhen_tuning.pair 0 / 1): +7-18 % on the long-K dot.proj family (C4 945 -> 802 us, 1360
  // TF/s), but slower on the short-K, store-bound shapes (the pair's epilogues run in lock step), so the
  // default takes pairs for K >= 1024 (dhen_tuning.pair_k; 512 measured slower) with at least 64 pair items
  // (split-K items included: +13 % on the C4 attention FFN weight gradients).
  {
    const int pair_k = tune().pair_k;
    const int mode = g_gemm_pair >= 0 ? g_gemm_pair : tune().pair;
    const int64_t pitems = (int64_t)((g.M + 2 * BM - 1) / (2 * BM)) * p.tiles_n * g.batch;
    p.pair = (BN >= 128 && (splits == 1 || mode == 1 || (splits > 1 && g.M >= 2 * BM)) && mode != 0 &&
              (mode == 1 ? g.M > BM : (pitems * splits >= 64 && g.K >= pair_k))) ? 1 : 0;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, &p.a, g.a, g.M, g.K, g.batch, BM)) return cudaErrorNotSupported;
  if (!make_map(&mb, &p.b, g.b, g.N, g.K, g.batch, p.pair ? BN / 2 : BN)) return cudaErrorNotSupported;
  if (p.pair) p.tiles_m = (g.M + 2 * BM - 1) / (2 * BM);
  g_last_gemm_pair = p.pair;
  p.n_fast = (p.tiles_n <= 16 && p.tiles_m >= p.tiles_n) ? 1 : 0;
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  p.splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;   // no empty splits
  p.ws = ws.ptr;
  p.trace = g_gemm_trace;
  p.pf_dist = tune().l2_prefetch;
  p.zbase = 0;
  p.nz = g.batch;
  p.lanes_rows = (g.c.cs != 1 && g.c.rs == 1 && splits == 1) ? 1 : 0;
  p.lean = (splits == 1 && make_lean(g, &p.ep)) ? 1 : 0;
  p.lean_id = p.lean ? lean_variant(p.ep.flags, p.ep.c_f32 != 0) : 0;
  const bool special = p.lean && (p.ep.flags & (EF_DCNB | EF_TRIU));
  p.fast8 = 0;
  if (p.lean && g.c.cs == 1 && g.N % 8 == 0) {
    auto al16 = [](const void* q) { return !q || ((uintptr_t)q % 16) == 0; };
    const View* vs[5] = {&g.c, &g.e.cross, &g.e.aux, &g.e.mask, &g.e.resid};
    bool ok = true;
    for (const View* v : vs)
      if (v->ptr && (!al16(v->ptr) || v->rs % 8 || v->bs0 % 8 || v->bs1 % 8 || v->rs_o % 8)) ok = false;
    if (g.e.triu_m) ok = true;   // scalar stores into the packed triangle
    p.fast8 = ok ? 1 : 0;
  }
  // specialised passes for the DCN-backward / triangle epilogues: row-major (fast8), or DCN backward with a
  // column-contiguous C (lanes on rows); anything else takes the generic epi_apply
  if (special && !(p.fast8 && p.lean_id > 0 && !p.lanes_rows) &&
      !((p.ep.flags & EF_DCNB) && p.lanes_rows && p.lean_id > 0)) { p.lean = 0; p.lean_id = 0; }
  p.fast = (!p.lanes_rows && splits == 1 && vec_ok(g.c) && vec_ok(g.e.cross) && vec_ok(g.e.aux) &&
            vec_ok(g.e.resid) && vec_ok(g.e.mask)) ? 1 : 0;
  if (special || g.e.triu_m || g.e.dcn_bwd) p.fast = 0;
  // TMA-store epilogue: row-major C (single-level rows, one batch stride), a variant within TS_FLAGS
  // (fp32 += as a TMA reduce-add), 128-B passes that fit the warp's column half
  OutMaps mc;
  memset(&mc, 0, sizeof mc);
  p.tstore = 0;
  {
    const int env = tune().tstore;
    const int es = g.c.dt == F32 ? 4 : 2;
    const int fl = p.lean ? p.ep.flags : -1;
    const bool flags_ok = fl >= 0 && (fl & ~TS_FLAGS) == 0 && (!(fl & EF_ACC) || g.c.dt == F32) && p.lean_id > 0;
    const bool geom_ok = g.c.cs == 1 && g.c.rdiv == 0 && (g.c.zdiv == 1 || g.c.bs1 == 0) && !p.lanes_rows &&
                         splits == 1 && ((uintptr_t)g.c.ptr % 16) == 0 && (g.c.rs * es) % 16 == 0 &&
                         (g.c.bs0 * es) % 16 == 0 && (g.c.dt == F32 || BN >= 128) && g.c.rs >= g.N;
    EncodeFn fn = encode_fn();
    if (env && flags_ok && geom_ok && fn) {
      const int64_t bstride = (g.batch > 1 && g.c.bs0) ? g.c.bs0 : (int64_t)g.c.rs * g.M;
      cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch};
      cuuint64_t strides[2] = {(cuuint64_t)(g.c.rs * es), (cuuint64_t)(bstride * es)};
      cuuint32_t box[3] = {(cuuint32_t)(128 / es), 32, 1}, estr[3] = {1, 1, 1};
      if (strides[1] % 16 == 0 && strides[1] > 0 &&
          fn(&mc.c, g.c.dt == F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g.c.ptr, dims,
             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        p.tstore = 1;
    }
  }
  // 3-D maps {N, M, batch} of a row-major view with 32 x 32 boxes (bf16: 64-B swizzle, fp32: 128-B) for the
  // operand epilogues below
  EncodeFn fn3 = encode_fn();
  auto map3 = [&](CUtensorMap* m, const View& v, bool f32) -> bool {
    const int es = f32 ? 4 : 2;
    if (!fn3 || !v.ptr || v.cs != 1 || v.rdiv || !(v.zdiv == 1 || v.bs1 == 0) || ((uintptr_t)v.ptr % 16) ||
        (v.rs * es) % 16 || v.rs < g.N)
      return false;
    const int64_t bstride = (g.batch > 1 && v.bs0) ? v.bs0 : (int64_t)v.rs * g.M;
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(v.rs * es), (cuuint64_t)(bstride * es)};
    cuuint32_t box[3] = {32, 32, 1}, estr[3] = {1, 1, 1};
    return strides[1] % 16 == 0 &&
           fn3(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, v.ptr, dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  const bool opnd_ok = p.lean && p.fast8 && !p.lanes_rows && !p.pair && splits == 1 && g.M % 32 == 0 && g.N % 32 == 0;
  // DCN-backward operand epilogue: X, A, dR in and dA, dX out as 32 x 32 boxes by TMA
  p.dcnt = 0;
  if (tune().dcn_tma && opnd_ok && (p.ep.flags & EF_DCNB) && g.M % BM == 0 && g.c.dt == F32) {
    const bool first = (p.ep.flags & EF_RESID) != 0;
    if (map3(&mc.x, g.e.cross, false) && map3(&mc.m, g.e.mask, false) && map3(&mc.a, g.e.aux, false) &&
        map3(&mc.c, g.c, true) && (!first || map3(&mc.r, g.e.resid, false)))
      p.dcnt = 1;
  }
  // DCN cross forward: X in, A (aux) and T (C) out as 32 x 32 bf16 boxes by TMA
  p.crosst = 0;
  if (tune().dcn_tma && opnd_ok && BN >= 128 && p.ep.flags == (EF_BIAS | EF_CROSS | EF_AUX) && g.c.dt == BF16 && !g.e.bias_gap_hi &&
      g.e.bias_dt == BF16 && p.lean_id > 0) {
    if (map3(&mc.x, g.e.cross, false) && map3(&mc.a, g.e.aux, false) && map3(&mc.c, g.c, false)) p.crosst = 1;
  }
  // fp32-residual epilogue (the token-map dgrad's first writer): dR in, C out as 32 x 32 boxes by TMA
  p.rst = 0;
  if (tune().resid_tma && opnd_ok && BN >= 128 && p.ep.flags == (EF_RESID | EF_R32) && g.c.dt == BF16 && p.lean_id > 0 &&
      g.e.resid.dt == F32) {
    if (map3(&mc.r, g.e.resid, true) && map3(&mc.c, g.c, false)) p.rst = 1;
  }
  p.lnst = 0;
  p.ln_rdiv = 0;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)p.a.mn_major << 15) | ((uint32_t)p.b.mn_major << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((p.pair ? 2 * BM : BM) >> 4) << 24);
  const int var = (p.lean_id > 0 && (p.fast8 || p.lanes_rows)) ? p.lean_id : 0;
  if (p.tstore && var != p.lean_id) p.tstore = 0;
  // LayerNorm epilogue with TMA: residual boxes in, R and Y boxes out over 4-D maps {N, L, M / L, batch}
  // (L = rows per group of a two-level row view, else M), 32-row warp boxes inside one group or whole groups
  if (tune().ln_tma && p.lean && (p.ep.flags & EF_LN) && var == p.lean_id && var > 0 && !p.lanes_rows && splits == 1 &&
      g.M % 32 == 0) {
    EncodeFn fn = encode_fn();
    const int L = g.c.rdiv ? g.c.rdiv : g.M;
    const bool geo = fn && g.M % L == 0 && (L % 32 == 0 || 32 % L == 0) && g.c.cs == 1 && (g.c.zdiv == 1 || g.c.bs1 == 0);
    auto map4 = [&](CUtensorMap* m, const View& v) -> bool {
      if (!v.ptr || v.dt != BF16 || ((uintptr_t)v.ptr % 16)) return false;
      const int64_t rs_o = g.c.rdiv ? v.rs_o : (int64_t)v.rs * L;
      const int64_t groups = g.M / L;
      const int64_t bstride = (g.batch > 1 && v.bs0) ? v.bs0 : rs_o * groups;
      cuuint64_t dims[4] = {(cuuint64_t)g.N, (cuuint64_t)L, (cuuint64_t)groups, (cuuint64_t)g.batch};
      cuuint64_t strides[3] = {(cuuint64_t)(v.rs * 2), (cuuint64_t)(rs_o * 2), (cuuint64_t)(bstride * 2)};
      for (int i = 0; i < 3; ++i)
        if (strides[i] % 16 || strides[i] == 0) return false;
      cuuint32_t box[4] = {64, (cuuint32_t)std::min(L, 32), (cuuint32_t)(L < 32 ? 32 / L : 1), 1}, estr[4] = {1, 1, 1, 1};
      return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
             CUDA_SUCCESS;
    };
    if (geo && map4(&mc.c, g.c) && map4(&mc.d, g.e.aux) && map4(&mc.r, g.e.resid)) {
      p.lnst = 1;
      p.ln_rdiv = L;
    }
  }
  // W-resident short-K GEMMs (Params::wr): the CTA's K x 256 weight tile stays in shared memory, the ring streams A
  const int fl_ = p.ep.flags;
  p.wr = (tune().wres && p.tstore && var > 0 && BN == 256 && !p.pair && splits == 1 && g.batch == 1 && p.kblocks <= 4 &&
          p.n_fast && (fl_ & ~TS_FLAGS) == 0 && !(fl_ & EF_ACC) && g.c.dt == BF16) ? 1 : 0;
  if (p.wr && tune().wres == 2 && g.M >= 4 * BM) {
    // the CTA-pair form: each CTA keeps half of the B tile, so the A ring is twice as deep (256-row pair tiles)
    Params q = p;
    q.pair = 1;
    if (make_map(&mb, &q.b, g.b, g.N, g.K, g.batch, BN / 2)) {
      p = q;
      p.tiles_m = (g.M + 2 * BM - 1) / (2 * BM);
      p.n_fast = (p.tiles_n <= 16 && p.tiles_m >= p.tiles_n) ? 1 : 0;
      if (!p.n_fast) p.wr = 0;
      p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)p.a.mn_major << 15) | ((uint32_t)p.b.mn_major << 16) |
                ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      g_last_gemm_pair = 1;
    } else {
      (void)make_map(&mb, &p.b, g.b, g.N, g.K, g.batch, BN);
    }
  }
  if (g.e.ln_gamma && (!p.lean || var != p.lean_id || (p.ep.flags & EF_LN) == 0 || p.lanes_rows)) return cudaErrorNotSupported;
  if (g.e.bits_mode && !p.tstore) return cudaErrorNotSupported;   // bitmask epilogues exist on the TMA-store path
  // column sums of the stored C exist on the bf16 TMA-store path only (rows = M / 32 blocks per batch item)
  if (g.e.csum && (!p.tstore || g.c.dt != BF16 || g.e.accumulate)) return cudaErrorNotSupported;
  // fused dA column sums exist in the row-major DCN-backward pass only (single CTAs, N <= 256)
  if (g.e.bsum && (!g.e.dcn_bwd || var == 0 || !p.fast8 || p.lanes_rows || p.pair || g.N > 256 ||
                   (p.ep.flags & EF_DCNB) == 0))
    return cudaErrorNotSupported;
  cudaError_t e = BN == 64 ? launch_bn64(p, ma, mb, mc, st, var) : BN == 128 ? launch_bn128(p, ma, mb, mc, st, var)
                                                               : launch_bn256(p, ma, mb, mc, st, var);
  if (e != cudaSuccess) return e;
  if (p.splits > 1) return splitk_reduce(g, p.splits, ws.ptr, st);
  return cudaSuccess;
}

}  // namespace dhen
