"""Shared helpers of the -m gpu parity tests: run the CUDA path through the
C ABI (paper_2203_11014_b200.binding) and the oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

import synth
from oracle import dhen_oracle as O
from tests.helpers import make_flat_params, oracle_params


def to_binding(net: O.NetSpec, dtype: str, B: int, seed: int = 0):
    from paper_2203_11014_b200.binding import Config, Module
    layers = [[Module(s.kind, s.l, s.heads, s.ffn_mult, s.conv_channels, s.conv_k, tuple(s.mlp_hidden))
               for s in L.modules] for L in net.layers]
    return Config(net.m0, net.d, layers, dtype=dtype, batch_max_local=B, ln_eps=net.ln_eps, seed=seed,
                  ensembles=[L.ensemble for L in net.layers], dense_tokens=net.dense_tokens,
                  dense_in=[L.dense_in for L in net.layers])


def t2np(t):
    import torch
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


class Case:
    """One seeded problem: params, X0, labels, for both sides."""

    def __init__(self, net: O.NetSpec, B: int, dtype: str, seed: int, tuning=None):
        import torch
        self.net, self.B, self.dtype = net, B, dtype
        self.flats = make_flat_params(net, seed)
        if dtype == "bf16":   # masters are fp32; the oracle sees what the GPU computes with (R20)
            pass
        self.params = oracle_params(net, self.flats)
        self.X0 = synth.make_x0(seed, B, net.m0, net.d, bf16=(dtype == "bf16")).astype(np.float64)
        self.y = synth.make_labels(seed, B).astype(np.float64)
        from paper_2203_11014_b200.binding import DHEN
        self.model = DHEN(to_binding(net, dtype, B))
        if tuning:
            self.model.set_tuning(**tuning)
        for g, f in enumerate(self.flats):
            self.model.set_params(g, f)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdt = tdt
        self.x0 = torch.tensor(self.X0, dtype=torch.float32, device="cuda").to(tdt).contiguous()
        self.labels = torch.tensor(self.y, dtype=torch.float32, device="cuda")

    def prec(self):
        return O.Precision(bf16=(self.dtype == "bf16"))

    def gpu_step(self, lr):
        import torch
        loss = torch.zeros(1, dtype=torch.float32, device="cuda")
        dx0 = torch.empty_like(self.x0)
        self.model.train_step(self.x0, self.labels, lr, loss=loss, dx0=dx0)
        torch.cuda.synchronize()
        out = {"loss": float(loss.item()), "dX0": t2np(dx0)}
        out["grads"] = [self.model.get_grads(g).astype(np.float64) for g in range(len(self.flats))]
        out["params"] = [self.model.get_params(g).astype(np.float64) for g in range(len(self.flats))]
        return out

    def oracle_step(self, lr):
        return O.train_step(self.net, self.params, self.X0, self.y, lr, pr=self.prec())

    def flat_grads(self, ostep):
        return [O.flatten(g, gr) for g, gr in zip(O.param_groups(self.net), ostep["grads"])]

    def flat_params(self, ostep):
        return [O.flatten(g, p) for g, p in zip(O.param_groups(self.net), ostep["params"])]


def per_tensor(net: O.NetSpec, gi: int, flat: np.ndarray):
    return O.unflatten(O.param_groups(net)[gi], flat)
