"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs (SURVEY §8(c) protocol).

G1  fp32 mode, full train step:   loss / dX0 / new params elem <= 1e-5, grads norm <= 1e-5.
G3  bf16 mode, full train step:   oracle emulates the bf16 storage points;
                                  norm <= 2e-2 for Y-side outputs and grads; ReLU-gated grads
                                  (a Linear feeding a ReLU) are report-only end to end (SURVEY G3':
                                  mask flips of near-zero pre-activations), bounded by a relative
                                  Frobenius error <= 0.5.
G2  bf16 layer-local:             oracle fed the GPU's own bf16 layer input and dY; every grad
                                  norm <= 2e-2 except the ReLU-gated ones, gated at the measured worst
                                  case 5e-2 (mask flips of pre-activations within rounding of 0;
                                  round 2 measured 0.045 on B200, profiles/r2_parity.txt).
Sizes span several 64/128 tiles plus ragged tails (B*m not a tile multiple); the timed launch
configurations (full per-GPU batch) are covered by sampled-sample parity (test_full_size_sampled).
Every comparison prints its achieved errors (run with -s)."""
import numpy as np
import pytest

from oracle import dhen_oracle as O
from tests.gpu_common import Case, per_tensor, t2np
from tests.helpers import M, config, elem_err, norm_err, small

pytestmark = pytest.mark.gpu

RELU_GATED_G2 = 5e-2   # measured worst case of the layer-local ReLU-gated gradients (see the docstring)


def _gated(name):
    """Weights / biases of a Linear that feeds a ReLU (SURVEY G3')."""
    return (".attn." in name and name.endswith(("W_1", "b_1"))) or \
        (".mlp." in name and name.endswith(("W_1", "b_1", "W_2", "b_2")))


def _frob(a, o):
    a, o = np.asarray(a, np.float64), np.asarray(o, np.float64)
    den = np.linalg.norm(o)
    return float(np.linalg.norm(a - o) / (den if den > 0 else 1.0))


def _compare(case, g, o, tol_elem, tol_norm, gated_report_only=False, label=""):
    """gated_report_only: ReLU-gated grads are reported (norm) and bounded by a relative Frobenius error
    <= 0.5 instead of gated at tol_norm (SURVEY G3', end-to-end bf16 only)."""
    net = case.net
    report = {}
    report["loss"] = abs(g["loss"] - o["loss"]) / max(1.0, abs(o["loss"]))
    report["dX0"] = norm_err(g["dX0"], o["dX0"])
    og = case.flat_grads(o)
    op = case.flat_params(o)
    worst, gated = [], []
    for gi in range(len(og)):
        gt = per_tensor(net, gi, g["grads"][gi])
        ot = per_tensor(net, gi, og[gi])
        for k in ot:
            e = norm_err(gt[k], ot[k])
            if gated_report_only and _gated(k):
                gated.append((e, _frob(gt[k], ot[k]), f"g{gi}.{k}"))
            else:
                worst.append((e, tol_norm, f"g{gi}.{k}"))
        report[f"params{gi}"] = elem_err(g["params"][gi], op[gi])
    bad = [(e, t, k) for e, t, k in worst if not e <= t] + [(f, 0.5, k) for _, f, k in gated if not f <= 0.5]
    top = sorted(worst, reverse=True)[:3]
    print(f"\nPARITY {label}: loss {report['loss']:.2e} dX0 {report['dX0']:.2e} "
          f"params {max(v for k, v in report.items() if k.startswith('params')):.2e} "
          f"worst grads " + ", ".join(f"{k} {e:.2e}" for e, _, k in top) +
          ("; ReLU-gated (report only) " + ", ".join(f"{k} norm {e:.2e} frob {f:.2e}" for e, f, k in
                                                     sorted(gated, reverse=True)[:4]) if gated else ""))
    msg = f"{report} worst grads {sorted(worst, reverse=True)[:5]} gated {gated}"
    assert report["loss"] <= tol_elem, msg
    assert report["dX0"] <= tol_norm, msg
    for gi in range(len(og)):
        assert report[f"params{gi}"] <= tol_elem, msg
    assert not bad, msg
    return report


@pytest.mark.parametrize("name,B", [("C1", 32), ("C1", 7), ("C2", 37), ("C3", 21), ("C4", 19), ("C5", 29)])
def test_fp32_train_step_matches_oracle(name, B):
    """G1: fp32 mode (exact FP32 FMA, no TF32) at 1e-5."""
    net = small(name)
    case = Case(net, B, "fp32", seed=2203011014 + 1)
    g = case.gpu_step(lr=0.1)
    o = case.oracle_step(lr=0.1)
    _compare(case, g, o, 1e-5, 1e-5, label=f"G1 fp32 {name} B={B}")


@pytest.mark.parametrize("name,B", [("C2", 37), ("C3", 21), ("C4", 19), ("C5", 29)])
def test_bf16_train_step_matches_oracle(name, B):
    """G3: bf16 storage, fp32 accumulation; oracle emulates the storage points."""
    net = small(name)
    case = Case(net, B, "bf16", seed=2203011014 + 2)
    g = case.gpu_step(lr=0.05)
    o = case.oracle_step(lr=0.05)
    _compare(case, g, o, 2e-2, 2e-2, gated_report_only=True, label=f"G3 bf16 small {name} B={B}")


def test_fp32_c1_full_config():
    """C1 exactly as BASELINE.json names it (1 layer {Dot 4, Linear 4}, 8 x 16, B = 32, fp32)."""
    case = Case(config("C1"), 32, "fp32", seed=2203011014 + 1)
    _compare(case, case.gpu_step(0.1), case.oracle_step(0.1), 1e-5, 1e-5, label="G1 C1 full")


@pytest.mark.parametrize("kind", ["dot", "attn", "conv", "dcn", "linear", "mlp"])
def test_bf16_layer_local(kind):
    """G2: one layer, the oracle fed the GPU's bf16 input and a fixed dY."""
    import torch
    m, d, B = 24, 32, 23
    s = M(kind, m if kind != "dot" else 16, heads=2, mlp_hidden=(96, 64))
    net = O.NetSpec(m, d, [O.LayerSpec([s] + ([M("linear", 8)] if kind == "dot" else []))])
    case = Case(net, B, "bf16", seed=77)
    mo = O.layer_dims(net)[0][1]
    y = torch.empty(B, mo, d, dtype=torch.bfloat16, device="cuda")
    case.model.zero_grad()
    case.model.layer_fwd(0, case.x0, y)
    rng = np.random.default_rng(5)
    dY = rng.standard_normal((B, mo, d)).astype(np.float32)
    dy = torch.tensor(dY, device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(case.x0)
    case.model.layer_bwd(0, dy, dx)
    torch.cuda.synchronize()
    pr = case.prec()
    P = O.compute_params(case.params, pr)[0]
    Yo, cache = O.layer_fwd(net, 0, case.X0, P, pr)
    dXo, go = O.layer_bwd(net, 0, cache, t2np(dy), P, pr)
    gg = per_tensor(net, 0, case.model.get_grads(0).astype(np.float64))
    errs = {"Y": elem_err(t2np(y), Yo), "dX": norm_err(t2np(dx), dXo)}
    errs.update({k: norm_err(gg[k], v) for k, v in go.items()})
    print(f"\nPARITY G2 {kind}: " + " ".join(f"{k} {e:.2e}" for k, e in errs.items()))
    bad = {k: e for k, e in errs.items() if e > (RELU_GATED_G2 if _gated(k) else 2e-2)}
    assert not bad, (bad, errs)


@pytest.mark.parametrize("dtype,m,d,k,path", [
    ("bf16", 16, 64, 3, "double-buffered whole-sample stencil (conv_db_k)"),
    ("bf16", 16, 24, 3, "whole-sample stencil (conv_sample_k, bf16: 2048 % d != 0)"),
    ("fp32", 16, 64, 3, "whole-sample stencil (conv_sample_k, fp32)"),
    ("bf16", 16, 64, 5, "row bands (conv_band_k / conv_wgrad_band_k, k = 5)"),
    ("fp32", 12, 24, 5, "row bands, fp32 (k = 5)"),
    ("fp32", 10, 16, 7, "generic per-element kernels (k = 7)"),
    ("bf16", 9, 16, 7, "generic per-element kernels, bf16 (k = 7)"),
])
def test_conv_kernel_family_matches_oracle(dtype, m, d, k, path):
    """Every conv kernel generation the dispatcher can pick (F7 / B7, Eq.(5)) against the oracle on one train step of
    a conv-only layer (+ a linear module so the conv is not the only dX writer): G1 fp32 1e-5, G3 bf16 2e-2."""
    net = O.NetSpec(m, d, [O.LayerSpec([M("conv", m // 2, conv_k=k, conv_channels=3), M("linear", m - m // 2)])])
    B = 11
    case = Case(net, B, dtype, seed=4242 + k)
    lr = 0.1 if dtype == "fp32" else 0.05
    g = case.gpu_step(lr)
    o = case.oracle_step(lr)
    tol = 1e-5 if dtype == "fp32" else 2e-2
    _compare(case, g, o, tol, tol, label=f"conv {dtype} m={m} d={d} k={k}: {path}")


def test_layer_bwd_accumulates_and_is_deterministic():
    """backward twice == 2 x backward once; bitwise repeatable."""
    import torch
    net = small("C4")
    case = Case(net, 11, "fp32", seed=3)
    m0, d = net.m0, net.d
    mo = O.layer_dims(net)[0][1]
    y = torch.empty(11, mo, d, device="cuda")
    dy = torch.randn(11, mo, d, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    dx = torch.empty_like(case.x0)
    case.model.zero_grad()
    case.model.layer_fwd(0, case.x0, y)
    case.model.layer_bwd(0, dy, dx)
    g1 = case.model.get_grads(0)
    case.model.layer_bwd(0, dy, dx)
    g2 = case.model.get_grads(0)
    assert np.array_equal(g2, 2 * g1) or np.abs(g2 - 2 * g1).max() <= 1e-6 * np.abs(g1).max()
    case.model.zero_grad()
    case.model.layer_fwd(0, case.x0, y)
    case.model.layer_bwd(0, dy, dx)
    assert np.array_equal(case.model.get_grads(0), g1)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_sampled(name):
    """Every bf16 config at its FULL per-GPU batch (C2 2048, C3 / C4 / C5 8192), i.e. the launch
    configurations bench.py times (pair / split-K / packing rules keyed on B): the logits and dL/dX0 of
    sampled samples against the oracle run on those samples alone (each depends on its own sample only;
    B_global = B scales dX0).  Sample 0, the last sample (ragged tail of every tile walk) and two inner ones."""
    import torch
    from paper_2203_11014_b200 import configs
    net = config(name)
    B = configs.BATCH[name]
    case = Case(net, B, "bf16", seed=2203011014 + 7)
    logits = torch.empty(B, dtype=torch.float32, device="cuda")
    case.model.forward(case.x0, logits)
    g = case.gpu_step(lr=0.01)
    assert np.isfinite(g["loss"]) and all(np.isfinite(x).all() for x in g["grads"])
    zl = logits.cpu().numpy().astype(np.float64)
    idx = [0, 1, B // 2 + 3, B - 1]
    o = O.train_step(net, case.params, case.X0[idx], case.y[idx], 0.0, B_global=B, pr=case.prec())
    e_z = np.abs(zl[idx] - o["logits"]).max() / max(1.0, np.abs(o["logits"]).max())
    e_dx = norm_err(g["dX0"][idx], o["dX0"])
    print(f"\nPARITY full-size {name} B={B} samples {idx}: logits {e_z:.2e} dX0 {e_dx:.2e}")
    assert e_z <= 2e-2 and e_dx <= 2e-2, (e_z, e_dx)


def test_full_size_c2_all_grads():
    """C2 at its full BASELINE batch (2048, the bench launch configuration): loss, dX0, every parameter
    gradient and every updated parameter against the oracle run on the whole batch (G3; C2 has no ReLU)."""
    net = config("C2")
    case = Case(net, 2048, "bf16", seed=2203011014 + 2)
    g = case.gpu_step(lr=0.01)
    o = case.oracle_step(lr=0.01)
    _compare(case, g, o, 2e-2, 2e-2, label="G3 full C2 B=2048")


@pytest.mark.parametrize("name,B,layers", [("C2", 40, 2), ("C3", 32, 4), ("C4", 16, 2), ("C5", 8, 8)])
def test_bf16_full_dims_train_step(name, B, layers):
    """G3 at BASELINE.json's per-layer shapes (m, d, l_i, heads, FFN, MLP widths) and a small batch
    that takes the same fused paths as the timed step (B a multiple of every 128 / l_i: the LayerNorm-
    fused packed token projections), so the contractions run on the tcgen05/TMA path exactly as in the
    bench (C4 truncated to 2 of its 8 identical layers to bound the fp64 oracle's memory).  ReLU-gated
    grads are chaotic end to end (mask flips of near-zero pre-activations, SURVEY G3'): reported and
    bounded here, gated layer-locally in test_bf16_full_dims_layer_local."""
    net = config(name)
    net = O.NetSpec(net.m0, net.d, net.layers[:layers])
    case = Case(net, B, "bf16", seed=2203011014 + 5)
    g = case.gpu_step(lr=0.01)
    o = case.oracle_step(lr=0.01)
    _compare(case, g, o, 2e-2, 2e-2, gated_report_only=True, label=f"G3 full-dims {name} B={B}")


@pytest.mark.parametrize("name,B,layers", [("C2", 24, 2), ("C3", 24, 4), ("C4", 16, 2), ("C5", 6, 8)])
def test_bf16_full_dims_layer_local(name, B, layers):
    """G2 for every layer at full per-layer shapes: run the stack layer by layer through the C ABI;
    the oracle gets the GPU's own bf16 layer input X_n and upstream gradient dY_n (emulating the
    same bf16 storage points) and must match Y_n, dX_n and every gradient of the layer at 2e-2
    (the ReLU-gated ones at the measured worst case RELU_GATED_G2)."""
    import torch
    net = config(name)
    net = O.NetSpec(net.m0, net.d, net.layers[:layers])
    case = Case(net, B, "bf16", seed=2203011014 + 6)
    dims = O.layer_dims(net)
    pr = case.prec()
    P = O.compute_params(case.params, pr)
    xs, x = [case.x0], case.x0
    case.model.zero_grad()
    for n, (mi, mo) in enumerate(dims):
        y = torch.empty(B, mo, net.d, dtype=torch.bfloat16, device="cuda")
        case.model.layer_fwd(n, x, y)
        xs.append(y)
        x = y
    rng = np.random.default_rng(11)
    dy = torch.tensor(rng.standard_normal((B, dims[-1][1], net.d)) / np.sqrt(B), dtype=torch.float32,
                      device="cuda").to(torch.bfloat16)
    dys = {}
    for n in reversed(range(len(dims))):
        dys[n] = dy
        dx = torch.empty_like(xs[n])
        case.model.layer_bwd(n, dy, dx)
        dy = dx
    torch.cuda.synchronize()
    for n in range(len(dims)):
        Yo, cache = O.layer_fwd(net, n, t2np(xs[n]), P[n], pr)
        dXo, go = O.layer_bwd(net, n, cache, t2np(dys[n]), P[n], pr)
        gg = per_tensor(net, n, case.model.get_grads(n).astype(np.float64))
        errs = {"Y": elem_err(t2np(xs[n + 1]), Yo)}
        if n > 0:
            errs["dX"] = norm_err(t2np(dys[n - 1]), dXo)
        errs.update({k: norm_err(gg[k], v) for k, v in go.items()})
        top = sorted(errs.items(), key=lambda kv: -kv[1])[:4]
        print(f"\nPARITY G2 full-dims {name} layer {n}: " + " ".join(f"{k} {e:.2e}" for k, e in top))
        bad = {k: e for k, e in errs.items() if e > (RELU_GATED_G2 if _gated(f".{k}") else 2e-2)}
        assert not bad, (n, bad, errs)


def test_graphed_step_matches_eager_bitwise():
    """dhen_train_step_graphed (CUDA graph replay) == dhen_train_step, bit for bit, over 3 steps."""
    import torch
    net = small("C4")
    outs = []
    for graphed in (False, True):
        case = Case(net, 13, "bf16", seed=99)
        loss = torch.zeros(1, device="cuda")
        losses = []
        for _ in range(3):
            if graphed:
                case.model.train_step_graphed(case.x0, case.labels, 0.05, loss=loss)
            else:
                case.model.train_step(case.x0, case.labels, 0.05, loss=loss)
            torch.cuda.synchronize()
            losses.append(loss.item())
        outs.append((losses, [case.model.get_params(g) for g in range(len(case.flats))]))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


def test_host_buffer_step_matches_device_step_bitwise():
    """dhen_train_step_host (pinned host inputs uploaded by the library on its copy stream, two staging slots,
    loss copied back to the host) == dhen_train_step on the same inputs, bit for bit, over 4 steps whose
    inputs alternate between two host batches -- with sync = 0 for the middle steps, so an upload overlaps the
    previous step."""
    import torch
    net = small("C4")
    B = 13
    outs = []
    for host in (False, True):
        case = Case(net, B, "bf16", seed=98)
        other = Case(net, B, "bf16", seed=97)   # a second batch (its model is not used)
        xs = [case.x0, other.x0]
        ys = [case.labels, other.labels]
        loss = torch.zeros(1, device="cuda")
        hx = [x.cpu().pin_memory() for x in xs]
        hy = [y.cpu().pin_memory() for y in ys]
        hl = [torch.zeros(1).pin_memory() for _ in range(4)]
        losses = []
        for k in range(4):
            if host:
                case.model.train_step_host(hx[k % 2], hy[k % 2], 0.05, loss_host=hl[k], sync=(k in (0, 3)))
            else:
                case.model.train_step(xs[k % 2], ys[k % 2], 0.05, loss=loss)
                torch.cuda.synchronize()
                losses.append(loss.item())
        torch.cuda.synchronize()
        if host:
            losses = [float(h.item()) for h in hl]
        outs.append((losses, [case.model.get_params(g) for g in range(len(case.flats))]))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("mods,m,d,B", [
    ([("dot", 128)], 128, 128, 6),                     # Dot alone: first AND last dX writer (dR in, bf16 dX out)
    ([("dot", 64), ("conv", 64)], 128, 128, 6),        # Dot first writer (dR in, fp32 accumulator out)
    ([("dcn", 64), ("dot", 64)], 128, 128, 6),         # Dot last writer (fp32 accumulator in, bf16 dX out)
    ([("dcn", 64), ("dot", 32), ("linear", 32)], 128, 256, 6),   # Dot in between (fp32 +=), C4 shape
])
def test_dot_gram_bwd_onchip_modes(mods, m, d, B):
    """B5's Gram backward with S built on chip (dot_bwd_tc.cu) in each of its four dX-writer forms, layer-local
    against the oracle (G2 protocol): the oracle gets the GPU's bf16 X and dY and emulates the storage points."""
    import torch
    net = O.NetSpec(m, d, [O.LayerSpec([M(k, l) for k, l in mods])])
    case = Case(net, B, "bf16", seed=404)
    mo = O.layer_dims(net)[0][1]
    y = torch.empty(B, mo, d, dtype=torch.bfloat16, device="cuda")
    case.model.zero_grad()
    case.model.layer_fwd(0, case.x0, y)
    rng = np.random.default_rng(9)
    dy = torch.tensor(rng.standard_normal((B, mo, d)) / np.sqrt(B), dtype=torch.float32,
                      device="cuda").to(torch.bfloat16)
    dx = torch.empty_like(case.x0)
    case.model.layer_bwd(0, dy, dx)
    torch.cuda.synchronize()
    pr = case.prec()
    P = O.compute_params(case.params, pr)[0]
    Yo, cache = O.layer_fwd(net, 0, case.X0, P, pr)
    dXo, go = O.layer_bwd(net, 0, cache, t2np(dy), P, pr)
    gg = per_tensor(net, 0, case.model.get_grads(0).astype(np.float64))
    errs = {"Y": elem_err(t2np(y), Yo), "dX": norm_err(t2np(dx), dXo)}
    errs.update({k: norm_err(gg[k], v) for k, v in go.items()})
    print(f"\nPARITY G2 dot-bwd on chip {mods}: " + " ".join(f"{k} {e:.2e}" for k, e in errs.items()))
    bad = {k: e for k, e in errs.items() if e > 2e-2}
    assert not bad, (bad, errs)


@pytest.mark.parametrize("name,dtype,B,tol,opt", [("C4", "fp32", 13, 1e-5, "adam"), ("C2", "bf16", 24, 2e-2, "adam"),
                                                  ("C4", "fp32", 13, 2e-4, "adam_bf16"), ("C2", "bf16", 24, 2e-2, "adam_bf16")])
def test_adam_steps_match_oracle(name, dtype, B, tol, opt):
    """NEXT#3 optimizer variant: dhen_config.optimizer = Adam (fp32 moments on the master shard, device step
    counter) over three training steps against the oracle's adam_update (pinned to torch.optim.Adam).  eps is
    1e-3 so the update is a smooth function of the gradient (at eps -> 0 Adam's first step is lr * sign(g),
    which turns rounding-level gradient differences into full-size parameter differences, SURVEY ledger 18).
    adam_bf16: the BF16 optimizer (R35), moments stored in bf16 on both sides; in fp32 mode the GPU rounds its fp32
    moments and the oracle its fp64 ones, so an element whose moment sits within fp32 error of a bf16 rounding
    boundary may land one bf16 ulp apart, moving that parameter by <= lr 2^-8 |m/sqrt(v)| (~4e-5 here): 2e-4."""
    import torch
    from tests.gpu_common import to_binding
    from tests.helpers import make_flat_params, oracle_params
    from paper_2203_11014_b200.binding import DHEN
    import synth
    net = small(name)
    lr, betas, eps = 0.01, (0.9, 0.99), 1e-3
    flats = make_flat_params(net, 31)
    cfg = to_binding(net, dtype, B)
    cfg.optimizer, cfg.adam = opt, (betas[0], betas[1], eps)
    model = DHEN(cfg)
    for gi, f in enumerate(flats):
        model.set_params(gi, f)
    X0 = synth.make_x0(32, B, net.m0, net.d, bf16=(dtype == "bf16")).astype(np.float64)
    y = synth.make_labels(32, B).astype(np.float64)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x0 = torch.tensor(X0, dtype=torch.float32, device="cuda").to(tdt)
    lab = torch.tensor(y, dtype=torch.float32, device="cuda")
    params = oracle_params(net, flats)
    st = O.adam_init(params)
    pr = O.Precision(bf16=(dtype == "bf16"))
    groups = O.param_groups(net)
    for step in range(3):
        model.train_step_graphed(x0, lab, lr)
        torch.cuda.synchronize()
        o = O.train_step(net, params, X0, y, 0.0, pr=pr)
        params, st = O.adam_update(params, o["grads"], st, lr, betas[0], betas[1], eps, bf16_state=(opt == "adam_bf16"))
        errs = [elem_err(model.get_params(gi), O.flatten(g, params[gi])) for gi, g in enumerate(groups)]
        print(f"\nPARITY {opt} {name} {dtype} step {step + 1}: params {max(errs):.2e}")
        assert max(errs) <= tol, (step, errs)


def _ens_net(ens, proj):
    l = 5 if proj else 12
    mods = [M("dot", l), M("dcn", l), M("attn", l, heads=2), M("conv", l), M("linear", l),
            M("mlp", l, mlp_hidden=(24, 20))]
    return O.NetSpec(12, 16, [O.LayerSpec(mods, ensemble=ens), O.LayerSpec([M("dcn", l), M("linear", l)], ensemble=ens)])


@pytest.mark.parametrize("ens", ["sum", "wsum"])
@pytest.mark.parametrize("proj", [False, True])
@pytest.mark.parametrize("dtype,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_ensemble_variants_match_oracle(ens, proj, dtype, tol):
    """NEXT#3 method variant: sum / weighted-sum ensembles of Eq.(1), every module kind, with and without
    the W_n shortcut, full train step against the oracle (G1 fp32 1e-5, G3 bf16 2e-2; the learnable ensemble
    weights are gradients like any other)."""
    net = _ens_net(ens, proj)
    case = Case(net, 24, dtype, seed=2203011014 + 9)
    g = case.gpu_step(lr=0.05)
    o = case.oracle_step(lr=0.05)
    _compare(case, g, o, tol, tol, gated_report_only=(dtype == "bf16"), label=f"ensemble {ens} proj={proj} {dtype}")


@pytest.mark.parametrize("dtype,tol,m,d,l,B", [("fp32", 1e-5, 12, 16, 6, 19), ("bf16", 2e-2, 12, 16, 6, 19),
                                               ("bf16", 2e-2, 64, 128, 32, 24)])
def test_dcn_literal_matches_oracle(dtype, tol, m, d, l, B):
    """NEXT#3 method variant: Eq.(7) read literally (R31: per-sample d x d Gram over tokens, u = G W + b) as a
    module next to the others, two layers, full train step against the oracle (G1 / G3)."""
    net = O.NetSpec(m, d, [O.LayerSpec([M("dcn_lit", l), M("dcn", m - l)]), O.LayerSpec([M("dcn_lit", l), M("linear", m - l)])])
    case = Case(net, B, dtype, seed=2203011014 + 11)
    g = case.gpu_step(lr=0.05)
    o = case.oracle_step(lr=0.05)
    _compare(case, g, o, tol, tol, label=f"paper-literal DCN {dtype} m={m} d={d}")


@pytest.mark.parametrize("dtype,tol,m,d,l,B", [("fp32", 1e-5, 8, 16, 4, 19), ("bf16", 2e-2, 8, 16, 4, 19),
                                               ("bf16", 2e-2, 16, 32, 8, 40)])
def test_dcn_full_matches_oracle(dtype, tol, m, d, l, B):
    """NEXT#3 method variant: the flattened full-rank DCN-v2 (R37: the cross on vec(X) with W in R^{md x md}) as a
    module next to the others, two layers (the second its dX's first and last writer), full train step against
    the oracle (G1 / G3)."""
    net = O.NetSpec(m, d, [O.LayerSpec([M("dcn_full", l), M("linear", m - l)]), O.LayerSpec([M("dcn_full", m)])])
    case = Case(net, B, dtype, seed=2203011014 + 12)
    g = case.gpu_step(lr=0.05)
    o = case.oracle_step(lr=0.05)
    _compare(case, g, o, tol, tol, label=f"flattened DCN {dtype} m={m} d={d}")


@pytest.mark.parametrize("dtype,tol,big", [("fp32", 1e-5, False), ("bf16", 2e-2, False), ("bf16", 2e-2, True)])
def test_dense_injection_matches_oracle(dtype, tol, big):
    """NEXT#3 method variant (R38): X0's first dense_tokens tokens injected into every module of the
    dense_in layers (the modules read [X_n ; D]; the shortcut and the LayerNorm X_n), dD summed over the layers into
    dX0's dense tokens -- full train step against the oracle (G1 / G3)."""
    if big:
        net = O.NetSpec(64, 128, [O.LayerSpec([M("dot", 32), M("dcn", 16), M("linear", 16)], dense_in=True),
                                  O.LayerSpec([M("attn", 32), M("mlp", 32, mlp_hidden=(256, 128))]),
                                  O.LayerSpec([M("dcn", 40), M("conv", 24)], dense_in=True)], dense_tokens=8)
        B = 32
    else:
        import sys
        sys.path.insert(0, "tests")
        from test_oracle_stack import _inj_net
        net, B = _inj_net(), 7
    case = Case(net, B, dtype, seed=2203011014 + 13)
    g = case.gpu_step(lr=0.05)
    o = case.oracle_step(lr=0.05)
    _compare(case, g, o, tol, tol, gated_report_only=(dtype == "bf16"), label=f"dense injection {dtype} big={big}")
