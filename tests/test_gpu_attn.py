"""The fused attention core (F4 forward / B6 core backward, csrc/attn_tc.cu) through the C ABI.

1. Against the fp64 oracle, layer-local (G2 protocol): an attention-only DHEN layer at the shapes the
   fused kernels cover (dh = 64 and 128, m = 128, a ragged m < 128, m = 1), the oracle fed the GPU's
   bf16 input and dY and emulating the bf16 storage points (P and dS rounded).
2. Against the library's own two-GEMM + softmax path (dhen_tuning.attn_fused = 0) on the same inputs:
   both round P, O, dS, dQKV to bf16 at the same points, so they agree far inside the 2e-2 gate.
"""
import numpy as np
import pytest

from oracle import dhen_oracle as O
from tests.gpu_common import Case, per_tensor, t2np
from tests.helpers import M, elem_err, norm_err

pytestmark = pytest.mark.gpu


def _layer(case, net, dY_seed=5):
    import torch
    B, d = case.B, net.d
    mo = O.layer_dims(net)[0][1]
    y = torch.empty(B, mo, d, dtype=torch.bfloat16, device="cuda")
    case.model.zero_grad()
    case.model.layer_fwd(0, case.x0, y)
    rng = np.random.default_rng(dY_seed)
    dy = torch.tensor(rng.standard_normal((B, mo, d)) / np.sqrt(B), dtype=torch.float32,
                      device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(case.x0)
    case.model.layer_bwd(0, dy, dx)
    torch.cuda.synchronize()
    return y, dy, dx, case.model.get_grads(0).astype(np.float64)


def _net(m, d, l=None):
    return O.NetSpec(m, d, [O.LayerSpec([M("attn", l or m, heads=2)])])


@pytest.mark.parametrize("m,d,B", [(128, 128, 24), (128, 256, 12), (100, 128, 20), (37, 256, 9), (1, 128, 200)])
def test_fused_attention_layer_matches_oracle(m, d, B):
    net = _net(m, d)
    case = Case(net, B, "bf16", seed=4242 + m)
    y, dy, dx, gg = _layer(case, net)
    pr = case.prec()
    P = O.compute_params(case.params, pr)[0]
    Yo, cache = O.layer_fwd(net, 0, case.X0, P, pr)
    dXo, go = O.layer_bwd(net, 0, cache, t2np(dy), P, pr)
    gt = per_tensor(net, 0, gg)
    errs = {"Y": elem_err(t2np(y), Yo), "dX": norm_err(t2np(dx), dXo)}
    errs.update({k: norm_err(gt[k], v) for k, v in go.items()})
    print(f"\nPARITY G2 attention m={m} d={d} B={B}: " +
          " ".join(f"{k} {e:.2e}" for k, e in sorted(errs.items(), key=lambda kv: -kv[1])[:5]))
    bad = {k: e for k, e in errs.items() if e > 2e-2}
    assert not bad, (bad, errs)


@pytest.mark.parametrize("m,d,B", [(128, 128, 300), (128, 256, 160), (100, 128, 300)])
def test_fused_attention_matches_two_gemm_path(m, d, B):
    """Same inputs through both attention-core paths (more items than SMs: persistent CTAs loop)."""
    net = _net(m, d)
    out = {}
    for mode in (0, 1):
        case = Case(net, B, "bf16", seed=99, tuning={"attn_fused": mode})
        y, dy, dx, gg = _layer(case, net)
        out[mode] = (t2np(y), t2np(dx), gg)
    (y0, dx0, g0), (y1, dx1, g1) = out[0], out[1]
    assert elem_err(y1, y0) <= 1e-2
    assert norm_err(dx1, dx0) <= 1e-2
    t0, t1 = per_tensor(net, 0, g0), per_tensor(net, 0, g1)
    for k in t0:
        tol = 5e-2 if k.endswith(("W_1", "b_1")) else 1e-2
        assert norm_err(t1[k], t0[k]) <= tol, (k, norm_err(t1[k], t0[k]))


def test_fused_attention_deterministic():
    """Bitwise-repeatable forward and backward (no atomics: one CTA per (sample, head))."""
    net = _net(128, 256)
    case = Case(net, 40, "bf16", seed=7)
    y1, _, dx1, g1 = _layer(case, net)
    y2, _, dx2, g2 = _layer(case, net)
    assert np.array_equal(t2np(y1), t2np(y2))
    assert np.array_equal(t2np(dx1), t2np(dx2))
    assert np.array_equal(g1, g2)


@pytest.mark.parametrize("m,d,B", [(128, 128, 200), (100, 256, 90)])
def test_layernorm_epilogue_matches_ln_kernel(m, d, B):
    """F5 / F6: LayerNorm fused into the out-projection / FFN2 GEMM epilogue (whole rows per tile) against
    the GEMM-into-fp32 + LayerNorm-kernel path on the same inputs (same bf16 storage points)."""
    net = _net(m, d)
    out = {}
    for mode in ("0", "1"):
        case = Case(net, B, "bf16", seed=123, tuning={"ln_fuse": int(mode)})
        y, dy, dx, gg = _layer(case, net)
        out[mode] = (t2np(y), t2np(dx), gg)
    (y0, dx0, g0), (y1, dx1, g1) = out["0"], out["1"]
    assert elem_err(y1, y0) <= 1e-2
    assert norm_err(dx1, dx0) <= 1e-2
    t0, t1 = per_tensor(net, 0, g0), per_tensor(net, 0, g1)
    for k in t0:
        tol = 5e-2 if k.endswith(("W_1", "b_1")) else 1e-2
        assert norm_err(t1[k], t0[k]) <= tol, (k, norm_err(t1[k], t0[k]))


@pytest.mark.parametrize("m,d,B", [(128, 128, 160), (100, 256, 70)])
def test_relu_bitmask_matches_bf16_mask(m, d, B):
    """B6 FFN: the ReLU derivative taken from the forward's bitmask (bit = stored bf16 F > 0, R22) gives the
    same data and weight gradients, bit for bit, as reading F itself.  (db_1's in-epilogue column sums exist
    on the bitmask's TMA-store path only, so both arms take the separate column-sum kernel here.)"""
    net = _net(m, d)
    out = {}
    for mode in ("0", "1"):
        case = Case(net, B, "bf16", seed=321, tuning={"fuse_db": 0, "relu_bits": int(mode)})
        y, dy, dx, gg = _layer(case, net)
        out[mode] = (t2np(y), t2np(dx), gg)
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
    assert np.array_equal(out["0"][2], out["1"][2])


@pytest.mark.parametrize("m,d,B", [(128, 128, 200), (100, 128, 300)])
def test_layernorm_epilogue_large_offset(m, d, B):
    """The fused LayerNorm epilogue's row statistics (chunked mean / M2, Chan-merged) on pre-norm rows with a
    large common offset (X0 = 1000 + N(0, 1): |mean| >> std): the same layer as the two-pass LayerNorm kernel
    path (ln_fuse = 0) within bf16 rounding; a one-pass E[v^2] - mean^2 form loses the variance here."""
    import torch
    net = _net(m, d)
    out = {}
    for mode in (0, 1):
        case = Case(net, B, "bf16", seed=55, tuning={"ln_fuse": mode})
        case.x0 = (case.x0.float() + 1000.0).to(torch.bfloat16).contiguous()
        y, dy, dx, gg = _layer(case, net)
        out[mode] = (t2np(y), t2np(dx))
    e_y, e_dx = elem_err(out[1][0], out[0][0]), norm_err(out[1][1], out[0][1])
    print(f"\nLN offset m={m}: Y {e_y:.2e} dX {e_dx:.2e}")
    assert e_y <= 2e-2 and e_dx <= 2e-2, (e_y, e_dx)
