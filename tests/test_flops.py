"""The MFU numerator (SURVEY §8(d) FLOP convention: forward contraction FLOPs 2·M·N·K, training = 3 x
forward) pinned to torch's FlopCounterMode, per module kind, for both the oracle's formula
(oracle.forward_flops_per_sample) and the product's twin (paper_2203_11014_b200/flops.py).

Each module's forward is written with torch LIBRARY routines in fp64 -- nn.TransformerEncoderLayer
(PyTorch semantics the paper's Eq.(4) reading R10 names), F.conv2d, F.linear, bmm -- and torch counts the
FLOPs of what actually ran.  Two documented differences from the convention, asserted exactly:
  * conv: torch counts the C unfolded filters, the convention the folded mean filter (Eq.(5) with the
    channel mean, R12), so torch = formula + (C - 1) · 2 · m · d · k²;
  * nothing else: the Gram is counted in full (torch's bmm), softmax / LN / elementwise are not counted.
SURVEY A.2's check: one C4 layer = 385.09 MF (formula 383.32 + unfolded conv 1.77)."""
import pytest
import torch
import torch.nn.functional as F
from torch.utils.flop_counter import FlopCounterMode

from oracle import dhen_oracle as O
from tests.helpers import M, config



@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def _module_forward(kind, s, m, d):
    """One sample through module kind `kind` (torch library ops), returning the unified [l, d] output."""
    X = torch.randn(1, m, d)
    l = s.l
    Wu = torch.randn(m, l)
    if kind == "dot":
        iu = torch.triu_indices(m, m, 1)
        G = torch.bmm(X, X.transpose(1, 2))[:, iu[0], iu[1]]
        return F.linear(G, torch.randn(l * d, G.shape[1])).reshape(1, l, d)
    if kind == "linear":
        return torch.matmul(Wu.t(), X)
    if kind == "dcn":
        A = F.linear(X, torch.randn(d, d), torch.randn(d))
        return torch.matmul(Wu.t(), X * A + X)
    if kind == "conv":
        k, C = s.conv_k, s.conv_channels
        T = F.conv2d(X[:, None], torch.randn(C, 1, k, k), padding=k // 2).mean(1)
        return torch.matmul(Wu.t(), T)
    if kind == "attn":
        enc = torch.nn.TransformerEncoderLayer(d, s.heads, s.ffn_mult * d, dropout=0.0, activation="relu",
                                               batch_first=True, norm_first=False)
        enc.train()
        # the math SDPA backend runs QK^T and PV as bmm (counted); the fused CPU kernel is not counted
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel(SDPBackend.MATH):
            return torch.matmul(Wu.t(), enc(X))
    if kind == "dcn_full":   # R37: the cross on the flattened sample
        x = X.reshape(1, m * d)
        A = F.linear(x, torch.randn(m * d, m * d), torch.randn(m * d))
        return torch.matmul(Wu.t(), (x * A + x).reshape(1, m, d))
    if kind == "dcn_lit":
        Xn = X.transpose(1, 2)
        return (torch.matmul(torch.bmm(Xn, Xn.transpose(1, 2)), torch.randn(d, l)).transpose(1, 2) + torch.randn(l, d))
    if kind == "mlp":
        h1, h2 = s.mlp_hidden
        a = F.relu(F.linear(X.reshape(1, m * d), torch.randn(h1, m * d), torch.randn(h1)))
        a = F.relu(F.linear(a, torch.randn(h2, h1), torch.randn(h2)))
        return F.linear(a, torch.randn(l * d, h2)).reshape(1, l, d)
    raise KeyError(kind)


def _counted(net):
    """torch-counted forward FLOPs of one sample through `net` (random weights: counts do not depend on them)."""
    d, tot = net.d, 0
    for (mi, mo), L in zip(O.layer_dims(net), net.layers):
        for s in L.modules:
            with FlopCounterMode(display=False) as fc:
                _module_forward(s.kind, s, mi, d)
            tot += fc.get_total_flops()
            if s.kind == "conv":   # the convention counts the folded (channel-mean) filter
                tot -= (s.conv_channels - 1) * 2 * mi * d * s.conv_k ** 2
        if mi != mo:               # Eq.(2) shortcut W_n^T X
            with FlopCounterMode(display=False) as fc:
                torch.matmul(torch.randn(mi, mo).t(), torch.randn(1, mi, d))
            tot += fc.get_total_flops()
    return tot


def _binding_cfg(net):
    from paper_2203_11014_b200.binding import Config, Module
    return Config(net.m0, net.d, [[Module(s.kind, s.l, s.heads, s.ffn_mult, s.conv_channels, s.conv_k,
                                          tuple(s.mlp_hidden)) for s in L.modules] for L in net.layers])


@pytest.mark.parametrize("kind", ["dot", "linear", "dcn", "conv", "attn", "mlp", "dcn_lit", "dcn_full"])
def test_module_flops_vs_torch_counter(kind):
    from paper_2203_11014_b200 import flops
    m, d = 12, 32
    s = M(kind, 5, heads=2, mlp_hidden=(48, 40))
    net = O.NetSpec(m, d, [O.LayerSpec([s])])          # 12 -> 5 tokens: the W_n shortcut is counted too
    c = _counted(net)
    assert O.forward_flops_per_sample(net) == c
    assert flops.forward_flops_per_sample(_binding_cfg(net)) == c


def test_c4_layer_survey_a2():
    """one full C4 layer, torch-counted with unfolded conv = 385.09 MF (formula 383.32)."""
    net = config("C4")
    one = O.NetSpec(net.m0, net.d, net.layers[:1])
    c = _counted(one)
    s_conv = one.layers[0].modules[2]
    unfolded = c + (s_conv.conv_channels - 1) * 2 * 128 * 256 * 9
    assert abs(unfolded / 1e6 - 385.09) < 0.01
    assert O.forward_flops_per_sample(one) == c
    assert abs(c / 1e6 - 383.32) < 0.01


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_config_flops_vs_torch_counter(name):
    """Whole BASELINE configs (C3 includes the 100 -> 128 W_n layer), both formulas."""
    from paper_2203_11014_b200 import configs, flops
    net = config(name)
    c = _counted(net)
    assert O.forward_flops_per_sample(net) == c
    assert flops.forward_flops_per_sample(configs.make(name)) == c
    assert flops.train_flops_per_sample(configs.make(name)) == 3 * c
