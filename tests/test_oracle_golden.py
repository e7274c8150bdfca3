"""SPEC hand examples as golden fixtures (tests/golden/spec_examples.json)."""
import json
import os

import numpy as np

from oracle import dhen_oracle as O
from tests.helpers import M

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_golden_dot():
    e = G["dot_orthogonal"]
    U, c = O.dot_fwd(np.array([e["X_tokens"]], float), {"W_m": np.array(e["W_m"], float)},
                     M("dot", e["l"]), O.FP64)
    assert c["Z"][0].tolist() == e["Z"] and U[0].tolist() == e["U"]
    e = G["dot_equal"]
    _, c = O.dot_fwd(np.array([e["X_tokens"]], float), {"W_m": np.ones((2, 1))}, M("dot", 1), O.FP64)
    assert c["Z"][0].tolist() == e["Z"]
    assert len(O.triu_pairs(G["dot_count"]["m"])[0]) == G["dot_count"]["h"]


def test_golden_linear_and_flops():
    e = G["linear_hand"]
    U, _ = O.linear_fwd(np.array([e["X_tokens"]], float), {"W": np.array(e["W"], float)}, M("linear", 1), O.FP64)
    assert U[0].tolist() == e["U"]
    e = G["linear_flops"]
    net = O.NetSpec(e["m"], e["d"], [O.LayerSpec([M("linear", e["l"])])])
    # the layer also maps 6 -> 4 tokens through W_n (2*6*4*8 = 384 more); the module part is 384
    assert O.forward_flops_per_sample(net) - 2 * e["m"] * e["l"] * e["d"] == e["flops"]


def test_golden_misc():
    Y, _, _ = O.ln_fwd(np.array([[G["layernorm_const"]["R"]]], float), np.ones(4), np.zeros(4), 1e-5)
    assert Y[0, 0].tolist() == G["layernorm_const"]["Y"]
    assert O._softmax_rows(np.array([[3.7]])).tolist() == G["softmax_len1"]["P"]
    s = O.sigmoid(0.0)
    assert s * (1 - s) == G["sigmoid_grad0"]["value"]
    assert O.sigmoid(0.0) == G["zero_head"]["prob"]
    e = G["concat_shortcut"]
    net = O.NetSpec(e["m_in"], 8, [O.LayerSpec([M("linear", e["l"][0]), M("dot", e["l"][1])])])
    assert dict((n, list(s)) for n, s, _ in O.param_groups(net)[0])["W_n"] == e["W_n"]
