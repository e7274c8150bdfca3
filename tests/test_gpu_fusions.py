"""A/B tests of a context's schedule / fusion switches (dhen_tuning, include/dhen_debug.h; per context, set
through dhen_set_tuning -- nothing is read from the environment): each variant must reproduce the default
schedule on the same inputs -- bit for bit where the arithmetic is the same, within bf16 rounding where a
fusion changes where a value is rounded.

overlap       weight gradients / module branches on a second stream           -> bitwise identical
defer_join    side-stream joins deferred to buffer reuse                      -> bitwise identical
trail         LayerNorm / head parameter sums trailing on the side stream     -> bitwise identical
bd_pre        every layer's block-diagonal token maps in one launch per step  -> bitwise identical
ln_fuse       LayerNorm in the producing GEMM epilogues (F5, F6, F12)         -> same storage points
first_writer  first / last dX writer (B3, B10) instead of LN-bwd init + cast  -> same fp32 sums, other order
relu_bits     FFN ReLU derivative from a bitmask                               -> bitwise identical
pair          CTA-pair GEMMs vs single-CTA tiles                               -> same sums up to split grouping
fuse_db       bias gradients from GEMM epilogue column sums (DCN db, FFN db_1) -> same values, other grouping
vdy           head dY formed inside the last LayerNorm backward (not stored)   -> bitwise identical
sym           dot backward: S on chip (-1) / dense S via a shared image (1, 2) / staged (0) -> bitwise identical
tstore        TMA-store GEMM epilogue vs the register epilogue                 -> same values (db_1 grouping)
ln_tma        LayerNorm epilogue: residual by TMA, R / Y by TMA store          -> bitwise identical
dcn_tma       DCN-backward epilogue: X / A / dR by TMA, dA / dX by TMA store   -> bitwise (db grouping)
dcn_fused     DCN backward as one kernel vs dT GEMM + dA W GEMM               -> bitwise (db grouping)
l2_prefetch   short-K GEMM operands prefetched into L2 items ahead (off)      -> bitwise identical
wres          short-K GEMMs with the weight tile resident in shared memory    -> bitwise identical
resid_tma     fp32-residual epilogue: dR by TMA boxes, C by TMA store         -> bitwise identical
"""
import numpy as np
import pytest

from oracle import dhen_oracle as O
from tests.gpu_common import Case, per_tensor
from tests.helpers import config, norm_err

pytestmark = pytest.mark.gpu


def _step(net, B, seed, tuning):
    case = Case(net, B, "bf16", seed=seed, tuning=tuning)
    return case.gpu_step(lr=0.01)


def _cmp(a, b, net, tol):
    if tol == 0:
        assert a["loss"] == b["loss"]
        assert np.array_equal(a["dX0"], b["dX0"])
        for ga, gb in zip(a["grads"], b["grads"]):
            assert np.array_equal(ga, gb)
        return
    assert abs(a["loss"] - b["loss"]) <= tol * max(1.0, abs(b["loss"]))
    assert norm_err(a["dX0"], b["dX0"]) <= tol
    for gi, (ga, gb) in enumerate(zip(a["grads"], b["grads"])):
        ta, tb = per_tensor(net, gi, ga), per_tensor(net, gi, gb)
        for k in tb:
            gated = k.endswith(("W_1", "b_1", "W_2", "b_2")) and (".mlp." in k or ".attn." in k)
            assert norm_err(ta[k], tb[k]) <= (5e-2 if gated else tol), (gi, k, norm_err(ta[k], tb[k]))


def _net(name, layers):
    net = config(name)
    return O.NetSpec(net.m0, net.d, net.layers[:layers])


@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2), ("C3", 32, 2), ("C5", 16, 2)])
def test_side_streams_bitwise(name, B, layers):
    net = _net(name, layers)
    a = _step(net, B, 11, {"overlap": 0})
    b = _step(net, B, 11, {"overlap": 1})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2), ("C5", 16, 2)])
def test_fused_layernorm_matches_kernel(name, B, layers):
    net = _net(name, layers)
    a = _step(net, B, 12, {"ln_fuse": 0})
    b = _step(net, B, 12, {"ln_fuse": 1})
    _cmp(a, b, net, 1e-2)


@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2), ("C5", 16, 2), ("C3", 32, 2)])
def test_first_last_dx_writer(name, B, layers):
    net = _net(name, layers)
    a = _step(net, B, 13, {"first_writer": 0})
    b = _step(net, B, 13, {"first_writer": 1})
    _cmp(a, b, net, 1e-2)


@pytest.mark.parametrize("name,B,layers", [("C2", 2048, 2), ("C4", 128, 2)])
def test_cta_pairs_match_single_cta(name, B, layers):
    """CTA-pair GEMMs (cta_group::2, deeper ring; LayerNorm epilogues included) against single-CTA tiles on
    the same step, at batch sizes where the size rule takes pairs (C2: the dot projection family at the
    bench's B = 2048; C4: FFN2 and the long-K weight gradients).  Same MMA chain per output row, so the
    results agree to rounding of the split-K reduction grouping."""
    net = _net(name, layers)
    a = _step(net, B, 14, {"pair": 0})
    b = _step(net, B, 14, {"pair": -1})
    _cmp(a, b, net, 1e-2)


@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C5", 16, 2), ("C3", 32, 2), ("C4", 16, 2)])
def test_fused_bias_grads(name, B, layers):
    """Bias gradients summed inside the producing GEMM epilogues against the separate column-sum kernel
    (same stored bf16 values, other grouping): B8 db = sum of dA (per-CTA partial rows from the DCN dT GEMM)
    and B6 db_1 = sum of dF (32-row partial rows from the FFN2 dgrad's TMA-store epilogue)."""
    net = _net(name, layers)
    a = _step(net, B, 15, {"fuse_db": 0})
    b = _step(net, B, 15, {"fuse_db": 1})
    _cmp(a, b, net, 1e-3)


@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2)])
def test_head_gradient_formed_in_ln_backward(name, B, layers):
    """B1 -> B2: the head's dY = bf16(dz_b / m w) formed inside the last layer's LayerNorm backward (never
    stored) is bit-identical to the head kernel writing it and the LayerNorm backward reading it."""
    net = _net(name, layers)
    a = _step(net, B, 16, {"vdy": 0})
    b = _step(net, B, 16, {"vdy": 1})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2)])
def test_dense_symmetrisation_bitwise(name, B, layers, mode):
    """B-dot: S = sym(dZ) scattered through a dense bf16 m x (m+2) shared image (one warp per triangle row)
    is bit-identical to the staged-triangle kernel (both copy the stored bf16 values); mode 1 stages the
    triangle in shared memory first, mode 2 reads it from global memory."""
    net = _net(name, layers)
    a = _step(net, B, 17, {"sym": 0})
    b = _step(net, B, 17, {"sym": int(mode)})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("switch", ["defer_join", "trail", "bd_pre", "tstore", "ln_tma", "wres", "resid_tma"])
@pytest.mark.parametrize("name,B,layers", [("C2", 64, 2), ("C4", 16, 2), ("C3", 32, 2)])
def test_schedule_switches_bitwise(name, B, layers, switch):
    """Schedule-only switches (same kernels' arithmetic in another order of launch / store path): the
    default and the switch turned off give bit-identical loss, dL/dX0 and gradients.  Without the TMA-store
    epilogue the FFN db_1 column sums come from the separate column-sum kernel (other grouping; the ReLU
    bitmask, a TMA-store feature, also falls back to the bf16 mask): 1e-3 there."""
    net = _net(name, layers)
    a = _step(net, B, 18, {switch: 0})
    b = _step(net, B, 18, {})
    _cmp(a, b, net, 1e-3 if switch == "tstore" else 0)


@pytest.mark.parametrize("wres", [1, 2])
@pytest.mark.parametrize("name,B,layers", [("C4", 256, 1), ("C3", 512, 1)])
def test_wres_many_items_bitwise(name, B, layers, wres):
    """W-resident GEMMs over many items a CTA (FFN1 / FFN2 dgrad / QKV at C4, the MLP GEMMs at C3), one CTA or a
    CTA pair a tile: bit-identical to the streamed-B kernel."""
    net = _net(name, layers)
    a = _step(net, B, 25, {"wres": 0})
    b = _step(net, B, 25, {"wres": wres})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("name,B,layers", [("C4", 256, 1), ("C5", 1024, 1)])
def test_l2_prefetch_bitwise(name, B, layers):
    """The producer's L2 prefetch of later items' operand tiles (dhen_tuning.l2_prefetch, off by default:
    measured slower) only moves data into L2: bit-identical steps.  Batches large enough that the
    short-K GEMMs have more than 2 x 148 items, so the prefetch is issued."""
    net = _net(name, layers)
    a = _step(net, B, 24, {"l2_prefetch": 2})
    b = _step(net, B, 24, {})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("name,B,layers", [("C4", 16, 2), ("C2", 64, 2)])
def test_ln_tma_cta_pairs_bitwise(name, B, layers):
    """The TMA LayerNorm epilogue in CTA-pair GEMMs (pair = 1 forces cta_group::2 tiles wherever expressible:
    the dot projection with its LayerNorm) against the register epilogue on the same pair tiles: bit-identical."""
    net = _net(name, layers)
    a = _step(net, B, 23, {"ln_tma": 0, "pair": 1})
    b = _step(net, B, 23, {"pair": 1})
    _cmp(a, b, net, 0)


def test_ln_tma_small_token_groups():
    """The TMA LayerNorm epilogue over two-level rows: a 16-token Linear module's packed token projection
    (8 samples per 128-row tile, 4-D boxes of 16 tokens x 2 samples) and a 48-token one (groups of 48 rows:
    not expressible as 32-row boxes, so the register epilogue runs) -- bit-identical to ln_tma = 0."""
    net = O.NetSpec(64, 128, [O.LayerSpec([O.ModuleSpec("linear", 16), O.ModuleSpec("dot", 48)]),
                              O.LayerSpec([O.ModuleSpec("linear", 64)])])
    a = _step(net, 32, 19, {"ln_tma": 0})
    b = _step(net, 32, 19, {})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("name,B,layers", [("C4", 16, 2)])
def test_gram_bwd_onchip_matches_dense_s(name, B, layers):
    """B5: the Gram backward with S built on chip from the packed dZ (sym = -1, dot_bwd_tc.cu) against the dense-S
    path (S scattered to HBM by the symmetrisation kernel, then a batched GEMM): the same MMA chain over the same
    bf16 operands (C2's two stacked samples add exact zeros), so loss, dX0 and every gradient agree bit for bit."""
    net = _net(name, layers)
    a = _step(net, B, 19, {"sym": 1})
    b = _step(net, B, 19, {})
    _cmp(a, b, net, 0)


@pytest.mark.parametrize("name,B,layers", [("C3", 32, 2), ("C4", 16, 2)])
def test_ffn_recompute_bitwise(name, B, layers):
    """NEXT#2 activation recompute (dhen_config.recompute = 1): the attention FFN hidden F is kept in one shared
    buffer and recomputed by the backward from the saved Z1 -- the same GEMM on the same operands, so loss,
    dX0 and every gradient are bit-identical, with less work memory."""
    from paper_2203_11014_b200 import binding
    from tests.gpu_common import to_binding
    net = _net(name, layers)
    a = _step(net, B, 20, {})
    cfg = to_binding(net, "bf16", B)
    cfg.recompute = 1
    case = Case(net, B, "bf16", seed=20)
    model = binding.DHEN(cfg)
    for g, f in enumerate(case.flats):
        model.set_params(g, f)
    case.model = model
    b = case.gpu_step(lr=0.01)
    _cmp(a, b, net, 0)
    assert binding.sizes(cfg)[1] < binding.sizes(to_binding(net, "bf16", B))[1]


@pytest.mark.parametrize("case_", ["C2", "C4", "C5", "wn"])
def test_dcn_tma_epilogue_matches_lane_epilogue(case_):
    """The dT GEMM's DCN-backward epilogue with TMA-staged operand boxes (dhen_tuning.dcn_tma = 1) against the
    per-lane global-load epilogue: the same per-element arithmetic (dA = bf16(dT X), dX = dT A + dT (+ dR), the
    non-first writer's fp32 add now a TMA reduce-add), so everything is bit-identical except the DCN bias
    gradient, whose column sums of the stored dA are grouped differently (fp32 rounding only)."""
    if case_ == "wn":
        net = O.NetSpec(128, 128, [O.LayerSpec([O.ModuleSpec("dcn", 64)]), O.LayerSpec([O.ModuleSpec("dcn", 64)])])
        B = 32
    else:
        B, layers = {"C2": (64, 2), "C4": (16, 2), "C5": (16, 2)}[case_]
        net = _net(case_, layers)
    a = _step(net, B, 22, {"dcn_tma": 0, "dcn_fused": 0})   # (the two-GEMM path, where the dT epilogue runs)
    b = _step(net, B, 22, {"dcn_tma": 1, "dcn_fused": 0})
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["dX0"], b["dX0"])
    for gi, (ga, gb) in enumerate(zip(a["grads"], b["grads"])):
        ta, tb = per_tensor(net, gi, ga), per_tensor(net, gi, gb)
        for k in tb:
            if k.endswith("dcn.b"):
                assert norm_err(ta[k], tb[k]) <= 1e-5, (gi, k)
            else:
                assert np.array_equal(ta[k], tb[k]), (gi, k, norm_err(ta[k], tb[k]))


@pytest.mark.parametrize("case_", ["C2", "C4", "C5", "wn"])
def test_dcn_fused_backward_matches_two_gemms(case_):
    """B8 as one kernel (dcn_bwd_tc.cu, the default: dT, dA, dA W with the partial dX kept in TMEM, W streamed, the
    operands and outputs as TMA boxes) against the two-GEMM path with the fp32 partial dX in HBM, on the same step:
    the same arithmetic in the same order, so loss, dX0 and every gradient are bit-identical -- except the DCN bias
    gradient, whose column sums of the stored dA are grouped differently (fp32 rounding only).  C2: two samples per
    tile; C4: separate dU / dA tiles (K1 = 32); C5: the shared-tile form (K1 = 128); 'wn': a 128 -> 64 token DCN
    layer (the W_n shortcut initialises the accumulator: fp32 base) followed by a two-samples-per-tile 64 -> 64 one."""
    if case_ == "wn":
        net = O.NetSpec(128, 128, [O.LayerSpec([O.ModuleSpec("dcn", 64)]), O.LayerSpec([O.ModuleSpec("dcn", 64)])])
        B = 32
    else:
        B, layers = {"C2": (64, 2), "C4": (16, 2), "C5": (16, 2)}[case_]
        net = _net(case_, layers)
    a = _step(net, B, 21, {"dcn_fused": 0})
    b = _step(net, B, 21, {"dcn_fused": 1})
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["dX0"], b["dX0"])
    for gi, (ga, gb) in enumerate(zip(a["grads"], b["grads"])):
        ta, tb = per_tensor(net, gi, ga), per_tensor(net, gi, gb)
        for k in tb:
            if k.endswith("dcn.b"):
                assert norm_err(ta[k], tb[k]) <= 1e-5, (gi, k)
            else:
                assert np.array_equal(ta[k], tb[k]), (gi, k, norm_err(ta[k], tb[k]))
