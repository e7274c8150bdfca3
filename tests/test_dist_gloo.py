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


# ----------------------------------------------------------------------------------------------------------
# Feature processing with column-sharded tables (NEXT#4, R36): the protocol the library runs over NCCL --
# the library's LPT shard plan (host-only C ABI), each rank pooling its shards for the global batch, the pooled
# all-to-all, X0 assembly, the reverse all-to-all of dX0's columns, the shard owners' sparse SGD and the bottom
# MLP's gradient all-reduce -- in fp64 numpy over gloo, against the unsharded oracle on the whole batch.
FP_ROWS, FP_D, FP_NDENSE, FP_HIDDEN, FP_NDTOK, FP_B = (300, 40, 1000, 7, 64), 128, 16, (32,), 2, 6


def _fp_case():
    import synth
    from oracle import fp_oracle as FO
    spec = FO.FPSpec(list(FP_ROWS), FP_NDENSE, list(FP_HIDDEN), FP_NDTOK, FP_D)
    P = FO.fp_init(spec, np.random.default_rng(9))
    Bg = WORLD * FP_B
    ids, off, dense = synth.make_fp_batch(9, Bg, list(FP_ROWS), FP_NDENSE, 5.0, bf16=False, empty_frac=0.1)
    G = np.random.default_rng(10).standard_normal((Bg, spec.m0, FP_D))
    return spec, P, ids.astype(np.int64), off.astype(np.int64), dense.astype(np.float64), G


def _fp_plan():
    import ctypes as C
    from paper_2203_11014_b200 import binding as B
    lib = B.load()
    r = (C.c_longlong * len(FP_ROWS))(*FP_ROWS)
    h = (C.c_int * len(FP_HIDDEN))(*FP_HIDDEN)
    cfg = B.dhen_fp_config(len(FP_ROWS), r, FP_NDENSE, len(FP_HIDDEN), h, FP_NDTOK, FP_D, B.FP32, FP_B, 1000, 0)
    S = (C.c_int * len(FP_ROWS))()
    own = (C.c_int * (len(FP_ROWS) * FP_D // 32))()
    assert lib.dhen_fp_shard_plan(C.byref(cfg), WORLD, S, own) == 0
    S = list(S)
    shards, g = [], 0   # (table, col0, width, owner)
    for t, s in enumerate(S):
        for k in range(s):
            shards.append((t, k * FP_D // s, FP_D // s, own[g]))
            g += 1
    return shards


def _fp_worker(rank, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from oracle import fp_oracle as FO
        spec, P, ids, off, dense, G = _fp_case()
        shards = _fp_plan()
        ns, nd, d, B = spec.n_sparse, spec.n_dtok, FP_D, FP_B
        Bg = WORLD * B
        mine = [s for s in shards if s[3] == rank]
        width = {r: sum(s[2] for s in shards if s[3] == r) for r in range(WORLD)}
        cmax = max(width.values())
        # forward: pool this rank's shards for every global sample -> the block of each sample's rank
        send = np.zeros((WORLD, B, cmax))
        for bg in range(Bg):
            o = 0
            for t, c0, w, _ in mine:
                bag = ids[off[bg * ns + t]:off[bg * ns + t + 1]]
                send[bg // B, bg % B, o:o + w] = FO.embedding_bag_sum(P["tables"][t][:, c0:c0 + w], bag)
                o += w
        recv = torch.zeros(WORLD * B * cmax, dtype=torch.float64)
        dist.all_to_all_single(recv, torch.tensor(send.reshape(-1)))
        recv = recv.numpy().reshape(WORLD, B, cmax)
        X0 = np.zeros((B, spec.m0, d))
        lo = rank * B
        h = dense[lo:lo + B]
        for W, b in zip(P["W"], P["b"]):   # data-parallel bottom MLP on this rank's samples
            h = np.maximum(h @ W.T + b, 0.0)
        X0[:, :nd] = h.reshape(B, nd, d)
        for r in range(WORLD):
            o = 0
            for t, c0, w, ow in shards:
                if ow != r:
                    continue
                X0[:, nd + t, c0:c0 + w] = recv[r, :, o:o + w]
                o += w
        # backward: dX0's columns of each shard to its owner, then the owner's sparse SGD over all samples
        lr = 0.3
        Gl = G[lo:lo + B]
        send2 = np.zeros((WORLD, B, cmax))
        for r in range(WORLD):
            o = 0
            for t, c0, w, ow in shards:
                if ow != r:
                    continue
                send2[r, :, o:o + w] = Gl[:, nd + t, c0:c0 + w]
                o += w
        recv2 = torch.zeros(WORLD * B * cmax, dtype=torch.float64)
        dist.all_to_all_single(recv2, torch.tensor(send2.reshape(-1)))
        recv2 = recv2.numpy().reshape(WORLD * B, cmax)   # row = global sample
        tables = {}
        o = 0
        for t, c0, w, _ in mine:
            T = P["tables"][t][:, c0:c0 + w].copy()
            g = np.zeros_like(T)
            for bg in range(Bg):
                for e in range(off[bg * ns + t], off[bg * ns + t + 1]):
                    g[ids[e]] += recv2[bg, o:o + w]
            tables[(t, c0)] = (T - lr * g).tolist()
            o += w
        # bottom MLP: local gradients, summed over ranks (the library's all-reduce), then SGD
        cache = {"H": [], "X0": X0, "B": B, "indices": np.zeros(0, np.int64), "offsets": np.zeros(B * 0 + 1, np.int64)}
        hh = dense[lo:lo + B]
        cache["H"].append(hh)
        for W, b in zip(P["W"], P["b"]):
            hh = np.maximum(hh @ W.T + b, 0.0)
            cache["H"].append(hh)
        spec0 = FO.FPSpec([], FP_NDENSE, list(FP_HIDDEN), nd, d)
        Pm = {"tables": [], "W": P["W"], "b": P["b"]}
        gr = FO.fp_bwd(spec0, Pm, cache, Gl[:, :nd + 0], FO.FPPrecision())
        mlp = []
        for a in gr["W"] + gr["b"]:
            t_ = torch.tensor(a)
            dist.all_reduce(t_)
            mlp.append(t_.numpy())
        L = len(P["W"])
        newW = [(P["W"][k] - lr * mlp[k]).tolist() for k in range(L)]
        newb = [(P["b"][k] - lr * mlp[L + k]).tolist() for k in range(L)]
        out_q.put((rank, X0.tolist(), tables, newW, newb))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_feature_processing():
    from paper_2203_11014_b200 import build
    from oracle import fp_oracle as FO
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fp_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(WORLD)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec, P, ids, off, dense, G = _fp_case()
    X0, cache = FO.fp_fwd(spec, P, ids, off, dense)
    newP = FO.fp_sgd(P, FO.fp_bwd(spec, P, cache, G), 0.3)
    shards = _fp_plan()
    assert len({s[3] for s in shards}) == WORLD   # both ranks own shards
    covered = {t: np.zeros(FP_D, bool) for t in range(len(FP_ROWS))}
    for rank, x0, tables, newW, newb in res:
        assert np.abs(np.array(x0) - X0[rank * FP_B:(rank + 1) * FP_B]).max() < 1e-12
        for (t, c0), T in tables.items():
            T = np.array(T)
            assert np.abs(T - newP["tables"][t][:, c0:c0 + T.shape[1]]).max() < 1e-12
            covered[t][c0:c0 + T.shape[1]] = True
        for k in range(len(newW)):
            assert np.abs(np.array(newW[k]) - newP["W"][k]).max() < 1e-12
            assert np.abs(np.array(newb[k]) - newP["b"][k]).max() < 1e-12
    assert all(c.all() for c in covered.values())   # every column of every table has exactly one owner's update
