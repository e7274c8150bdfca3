"""Training-FLOP accounting for MFU (SURVEY §8(d) convention, A18 / P:232
"Training FLOPs"): forward contraction FLOPs 2·M·N·K per GEMM (Gram counted
in full, conv with the folded kernel, elementwise / LN / softmax excluded),
training = 3 × forward.  Independent of the oracle's formula; both are pinned
to torch's FlopCounterMode in tests/test_flops.py."""
from __future__ import annotations


def forward_flops_per_sample(cfg) -> int:
    """cfg: binding.Config."""
    d = cfg.d
    tot = 0
    for (mi, mo), L in zip(cfg.dims(), cfg.layers):
        for s in L:
            l = s.l
            tok = 2 * mi * l * d                  # unify map W ∈ R^{m×l} (Eq.(4)-(6))
            if s.kind == "dot":
                h = mi * (mi - 1) // 2
                tot += 2 * mi * mi * d + 2 * h * l * d
            elif s.kind == "linear":
                tot += tok
            elif s.kind == "dcn_lit":
                tot += 2 * d * d * mi + 2 * d * d * l     # per-sample d x d Gram + projection (Eq.(7) literal)
            elif s.kind == "dcn":
                tot += 2 * mi * d * d + tok
            elif s.kind == "dcn_full":
                tot += 2 * (mi * d) ** 2 + tok          # the cross over the flattened sample (R37)
            elif s.kind == "conv":
                tot += 2 * mi * d * s.conv_k ** 2 + tok
            elif s.kind == "attn":
                f = s.ffn_mult * d
                tot += 6 * mi * d * d + 4 * mi * mi * d + 2 * mi * d * d + 4 * mi * d * f + tok
            elif s.kind == "mlp":
                h1, h2 = s.mlp_hidden
                tot += 2 * mi * d * h1 + 2 * h1 * h2 + 2 * h2 * l * d
        if mi != mo:
            tot += 2 * mi * mo * d
    return tot


def train_flops_per_sample(cfg) -> int:
    return 3 * forward_flops_per_sample(cfg)
