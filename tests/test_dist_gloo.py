"""Multi-process (world size 2, gloo, CPU) checks of the data-parallel / FSDP semantics the
library's NCCL path implements:

* each rank trains on its half of the global batch with the loss scaled by 1/B_global (R21);
* summing the per-rank gradients (the reduce-scatter + all-gather the library does per layer group)
  reproduces the single-process full-batch gradients, loss and SGD update;
* the library's host-side shard map (dhen_group_numel with world = 2) gives every rank the same shard
  size and world * shard covers the group.
The per-rank arithmetic is the fp64 oracle; the collectives are torch.distributed (gloo)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dhen_oracle as O
from tests.helpers import make_flat_params, oracle_params, small

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, name, B, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        net = small(name)
        params = oracle_params(net, make_flat_params(net, 21))
        rng = np.random.default_rng(7)
        X0 = rng.standard_normal((B, net.m0, net.d))
        y = (rng.random(B) < 0.3).astype(np.float64)
        lo, hi = rank * B // WORLD, (rank + 1) * B // WORLD
        o = O.train_step(net, params, X0[lo:hi], y[lo:hi], lr=0.1, B_global=B)
        groups = O.param_groups(net)
        # gradient reduction across ranks (what RS + AG of every group produce)
        red = []
        for gi, g in enumerate(groups):
            flat = torch.tensor(O.flatten(g, o["grads"][gi]))
            dist.all_reduce(flat)
            red.append(flat.numpy())
        loss = torch.tensor([o["loss"]])
        dist.all_reduce(loss)
        dx0 = torch.zeros(B, net.m0, net.d, dtype=torch.float64)
        dx0[lo:hi] = torch.tensor(o["dX0"])
        dist.all_reduce(dx0)
        # SGD on this rank's shard of every group, then all-gather the shards
        new = []
        for gi, g in enumerate(groups):
            p0 = O.flatten(g, params[gi])
            n = p0.size
            shard = (n + WORLD - 1) // WORLD
            pad = np.zeros(shard * WORLD)
            pad[:n] = p0
            gpad = np.zeros(shard * WORLD)
            gpad[:n] = red[gi]
            mine = torch.tensor(pad[rank * shard:(rank + 1) * shard] - 0.1 * gpad[rank * shard:(rank + 1) * shard])
            parts = [torch.zeros_like(mine) for _ in range(WORLD)]
            dist.all_gather(parts, mine)
            new.append(torch.cat(parts).numpy()[:n])
        # library shard map (host-only C ABI call; no GPU needed)
        from paper_2203_11014_b200 import binding
        from tests.gpu_common import to_binding
        cfg = to_binding(net, "bf16", B // WORLD)
        shards = [binding.group_numel(cfg, gi, binding.make_dist(rank, WORLD))[1] for gi in range(len(groups))]
        sh = torch.tensor(shards, dtype=torch.int64)
        sh_all = [torch.zeros_like(sh) for _ in range(WORLD)]
        dist.all_gather(sh_all, sh)
        out_q.put((rank, float(loss.item()), [r.tolist() for r in red], dx0.numpy().tolist(),
                   [x.tolist() for x in new], [s.tolist() for s in sh_all], shards))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_two_rank_step_equals_single_rank(name):
    from paper_2203_11014_b200 import build
    build.build()
    B = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, B, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(WORLD)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    net = small(name)
    params = oracle_params(net, make_flat_params(net, 21))
    rng = np.random.default_rng(7)
    X0 = rng.standard_normal((B, net.m0, net.d))
    y = (rng.random(B) < 0.3).astype(np.float64)
    full = O.train_step(net, params, X0, y, lr=0.1)
    groups = O.param_groups(net)
    for rank, loss, red, dx0, new, sh_all, shards in res:
        assert abs(loss - full["loss"]) < 1e-12
        assert np.abs(np.array(dx0) - full["dX0"]).max() < 1e-12
        for gi, g in enumerate(groups):
            ref = O.flatten(g, full["grads"][gi])
            assert np.abs(np.array(red[gi]) - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
            refp = O.flatten(g, full["params"][gi])
            assert np.abs(np.array(new[gi]) - refp).max() <= 1e-12
        # every rank sees the same shard sizes and world * shard covers each group
        assert sh_all[0] == sh_all[1]
        for gi, g in enumerate(groups):
            assert shards[gi] * WORLD >= O.group_size(g) and shards[gi] % 64 == 0
