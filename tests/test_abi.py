"""C ABI checks that need no GPU: the library loads, exports every symbol
include/dhen.h and include/dhen_debug.h declare, validates configs with the documented errors, and its
parameter layout agrees with the oracle's canonical order (sizes per group)."""
import os
import re

import pytest

from oracle import dhen_oracle as O
from tests.helpers import config, small

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def B():
    from paper_2203_11014_b200 import binding, build
    build.build()
    binding.load()
    return binding


def header_symbols(name="dhen.h"):
    src = open(os.path.join(ROOT, "include", name)).read()
    return sorted(set(re.findall(r"\b(dhen_[a-z_]+)\s*\(", src)))


def test_exports_every_header_symbol(B):
    lib = B.load()
    syms = header_symbols()
    dbg = header_symbols("dhen_debug.h")
    assert len(syms) >= 14 and len(dbg) >= 4
    assert not set(syms) & set(dbg)
    for s in syms + dbg:
        assert hasattr(lib, s), s
    assert set(syms) | set(dbg) == set(B.EXPORTS)


def _cfg(B, net, dtype="bf16", bmax=8):
    from tests.gpu_common import to_binding
    return to_binding(net, dtype, bmax)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_group_sizes_match_oracle_layout(B, name):
    net = config(name)
    cfg = _cfg(B, net)
    groups = O.param_groups(net)
    for gi, g in enumerate(groups):
        n, sh = B.group_numel(cfg, gi)
        assert n == O.group_size(g), (gi, n, O.group_size(g))
        assert sh >= n and sh % 64 == 0
    # sharded: shard * world covers the padded group
    d = B.make_dist(rank=1, world=8)
    for gi in range(len(groups)):
        n, sh = B.group_numel(cfg, gi, d)
        assert sh * 8 >= n and sh % 64 == 0


def test_validate_errors(B):
    bad = [
        (O.NetSpec(1, 16, [O.LayerSpec([O.ModuleSpec("dot", 2)])]), "Dot needs m >= 2"),
        (O.NetSpec(4, 12, [O.LayerSpec([O.ModuleSpec("linear", 2)])]), "multiple of 8"),
        (O.NetSpec(4, 24, [O.LayerSpec([O.ModuleSpec("attn", 2, heads=5)])]), "heads"),
        (O.NetSpec(4, 16, [O.LayerSpec([O.ModuleSpec("conv", 2, conv_k=4)])]), "odd"),
        (O.NetSpec(4, 16, [O.LayerSpec([O.ModuleSpec("linear", 0)])]), "l=0"),
    ]
    for net, frag in bad:
        with pytest.raises(B.DhenError) as ei:
            B.validate(_cfg(B, net))
        assert ei.value.status == 1 and frag in str(ei.value), str(ei.value)
    B.validate(_cfg(B, small("C4")))


def test_sizes_scale_with_batch(B):
    net = config("C2")
    s1, w1 = B.sizes(_cfg(B, net, bmax=64))
    s2, w2 = B.sizes(_cfg(B, net, bmax=128))
    assert s1 == s2 and w2 > w1
    # saved activations at C4's per-GPU batch fit one B200 (180 GB)
    s, w = B.sizes(_cfg(B, config("C4"), bmax=8192))
    assert s + w < 170e9, (s, w)


@pytest.mark.parametrize("ens", ["sum", "wsum"])
def test_ensemble_group_sizes_match_oracle(B, ens):
    """Sum / weighted-sum ensembles: the library's canonical group sizes (ensemble weights between the
    modules and W_n) equal the oracle's, and the 6 -> 5 token count (m_out = l) brings W_n."""
    mods = [O.ModuleSpec("dot", 5), O.ModuleSpec("dcn", 5), O.ModuleSpec("linear", 5)]
    net = O.NetSpec(6, 8, [O.LayerSpec(mods, ensemble=ens), O.LayerSpec(mods, ensemble=ens)])
    cfg = _cfg(B, net)
    for gi, g in enumerate(O.param_groups(net)):
        n, _ = B.group_numel(cfg, gi)
        assert n == O.group_size(g)
    assert O.layer_dims(net) == [(6, 5), (5, 5)]


def test_dense_injection_group_sizes_match_oracle(B):
    """Dense-token injection (R38): module parameters are shaped by m_in + dense_tokens in the injected layers
    (token maps, the Dot pairs, the MLP input, the flattened DCN) -- the library's group sizes equal the oracle's;
    a layer that injects with dense_tokens = 0 is rejected."""
    import sys
    sys.path.insert(0, "tests")
    from test_oracle_stack import _inj_net
    net = _inj_net()
    cfg = _cfg(B, net)
    for gi, g in enumerate(O.param_groups(net)):
        n, _ = B.group_numel(cfg, gi)
        assert n == O.group_size(g), gi
    bad = O.NetSpec(6, 8, [O.LayerSpec([O.ModuleSpec("dcn", 6)], dense_in=True)])
    with pytest.raises(B.DhenError) as e:
        B.validate(_cfg(B, bad))
    assert "dense_tokens" in str(e.value)


def test_ensemble_validation_errors(B):
    mods = [O.ModuleSpec("dot", 5), O.ModuleSpec("dcn", 4)]
    net = O.NetSpec(6, 8, [O.LayerSpec(mods, ensemble="sum")])
    with pytest.raises(B.DhenError) as e:
        B.validate(_cfg(B, net))
    assert "equal l_i" in str(e.value) or "sum ensemble" in str(e.value)


def test_fp_param_numel_and_validation(B):
    """Feature processing layer (NEXT#4) host-side layout: tables then (W_k, b_k) pairs; invalid configs
    are rejected without touching a device."""
    import ctypes as C
    lib = B.load()
    rows = (C.c_longlong * 2)(10, 20)
    hid = (C.c_int * 1)(32)
    cfg = B.dhen_fp_config(2, rows, 13, 1, hid, 2, 128, B.BF16, 64, 1000, 0)
    assert [lib.dhen_fp_param_numel(C.byref(cfg), w) for w in range(6)] == [1280, 2560, 32 * 13, 32, 256 * 32, 256]
    assert lib.dhen_fp_param_numel(C.byref(cfg), 6) == -1
    bad = B.dhen_fp_config(2, rows, 13, 1, hid, 2, 130, B.BF16, 64, 1000, 0)    # 4 does not divide d
    assert lib.dhen_fp_param_numel(C.byref(bad), 0) == -1
    h = C.c_void_p()
    assert lib.dhen_fp_init(C.byref(bad), None, C.byref(h)) == 1 and not h.value
    assert b"d = 130" in lib.dhen_last_error()


def test_fp_shard_plan_lpt(B):
    """The column-shard plan (R36), host only: a table larger than half of a rank's share is cut into
    power-of-two column shards of >= 32 columns, every shard has one owner, and LPT keeps every rank's load
    within one largest shard of the average (the greedy bound); one rank keeps every table whole."""
    import ctypes as C
    lib = B.load()
    rows = [1_000_000, 200_000, 50_000, 50_000, 3_000, 10, 900_000, 120_000]
    d = 256
    r = (C.c_longlong * len(rows))(*rows)
    cfg = B.dhen_fp_config(len(rows), r, 8, 0, None, 1, d, B.BF16, 64, 1000, 0)
    for world in (1, 2, 4, 8):
        S = (C.c_int * len(rows))()
        own = (C.c_int * (len(rows) * d // 32))()
        assert lib.dhen_fp_shard_plan(C.byref(cfg), world, S, own) == 0
        S = list(S)
        assert all(s & (s - 1) == 0 and d // s >= 32 for s in S)
        owners = list(own)[:sum(S)]
        assert all(0 <= o < world for o in owners)
        if world == 1:
            assert S == [1] * len(rows) and owners == [0] * len(rows)
            continue
        share = sum(rows) * d / world
        cost, load = [], [0.0] * world
        k = 0
        for t, s in enumerate(S):
            if rows[t] * d / s > share / 2:
                assert d // (2 * s) < 32   # only when a further cut would drop below 32 columns
            for _ in range(s):
                c = rows[t] * d / s
                cost.append(c)
                load[owners[k]] += c
                k += 1
        assert max(load) <= share + max(cost) + 1e-6
