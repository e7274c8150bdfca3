"""DHEN training-step benchmark (BASELINE.json metric: train samples/s, fwd + bwd).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A step is one `dhen_train_step` (forward of every layer, head + BCE loss,
backward, reduce-scatter when N > 1, SGD) over one synthetic batch of the
config's per-GPU size.  Default workload: C4, the north-star 8-layer
full-module DHEN (BASELINE configs[3]) at its per-GPU shard of 8192 samples.
N > 1 runs one process per GPU, batch-sharded with fully sharded parameters
(weak scaling: per-GPU batch fixed; N = 8 is configs[3]'s global 65536): under
torchrun the ranks come from the environment, otherwise `--gpus N` re-launches
itself through torch.distributed.run with N local ranks.

value:   device time (CUDA events on the launch stream) of K steps, inputs
         resident in HBM, L2 flushed (256 MiB write) before every timed step,
         max over ranks;  samples/s = N * B_local * K / time.
e2e:     the same through the C ABI's host-buffer entry (dhen_train_step_host)
         with pinned HOST buffers: every step copies X0 + labels host->device
         and the loss device->host inside the timed region (--fp: torch copies
         of ids / offsets / dense features around the device-pointer calls).
roofline: the op with the largest device time in a separate profiled pass of K
         steps (per-op CUDA events from dhen_profile), algorithmic FLOPs or bytes
         per launch / its mean launch time, against MEASURED_PEAKS.json.
cpu_baseline: the fp64 oracle (test infrastructure) on a bounded sample of the
         same workload on this host's cores (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm": j["hbm_gbs"], "tc": j["bf16_tflops"], "tc_sus": j["bf16_tflops_sustained"],
                "sm_max_mhz": j.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm": 6650.0, "tc": 1590.0, "tc_sus": 1400.0, "sm_max_mhz": 1965.0, "src": "fallback"}


class ClockSampler:
    """SM clock + throttle reasons polled through NVML every 2 ms during the timed region (the region of a
    short step can be far shorter than nvidia-smi's 200 ms interval); nvidia-smi CSV as a fallback."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, gpu: int):
        self.gpu, self.sm, self.reasons, self.max_mhz = gpu, [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis else self.gpu
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
            self.N = None
        return self

    def _poll(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS:
                    if r & getattr(N, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.N is not None:
            self.th.join(timeout=1)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "samples": len(self.sm),
                "source": "nvml", "reasons": sorted(self.reasons)}


def cpu_baseline(cfg_name: str, target_s: float = 8.0):
    """The fp64 oracle (as it stands) on a bounded sample of the workload, with all of the host's BLAS
    threads and again with one (1-thread and all-core samples/s)."""
    import numpy as np
    import synth
    from oracle import dhen_oracle as O
    from tests.helpers import config, make_flat_params, oracle_params
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        cores = max([t.get("num_threads", 1) for t in threadpool_info()] or [1])
    except Exception:
        threadpool_limits = None
        cores = os.cpu_count() or 1
    net = config(cfg_name)
    params = oracle_params(net, make_flat_params(net, 1))
    Bo = {"C1": 32, "C2": 16, "C3": 4, "C4": 2, "C5": 8}[cfg_name]
    X0 = synth.make_x0(1, Bo, net.m0, net.d, bf16=True).astype(np.float64)
    y = synth.make_labels(1, Bo).astype(np.float64)

    def timed():
        t0 = time.perf_counter()
        steps = 0
        while True:
            O.train_step(net, params, X0, y, 0.01)
            steps += 1
            el = time.perf_counter() - t0
            if el >= target_s or (steps >= 1 and el * (steps + 1) / steps > 3 * target_s):
                return steps, el
    steps, el = timed()
    out = {"value": steps * Bo / el, "unit": "samples/s", "cores": int(cores), "kind": "oracle",
           "sample": f"{steps} fp64 oracle train steps of {Bo} samples of {cfg_name} "
                     f"({el:.1f} s; cost is linear in B)", "seconds": round(el, 2)}
    if threadpool_limits is not None and cores > 1:
        with threadpool_limits(limits=1):
            s1, e1 = timed()
        out["one_thread"] = {"value": s1 * Bo / e1, "cores": 1, "seconds": round(e1, 2),
                             "sample": f"{s1} steps of {Bo} samples, BLAS limited to 1 thread"}
    return out


def run_reference(args):
    """--impl reference: the oracle is this tier's reference arm (host cores)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import synth
    from oracle import dhen_oracle as O
    from tests.helpers import config, make_flat_params, oracle_params
    net = config(args.config)
    params = oracle_params(net, make_flat_params(net, 1))
    Bo = {"C1": 32, "C2": 8, "C3": 2, "C4": 1, "C5": 4}[args.config]
    X0 = synth.make_x0(1, Bo, net.m0, net.d, bf16=True).astype(np.float64)
    y = synth.make_labels(1, Bo).astype(np.float64)
    for _ in range(args.warmup):
        O.train_step(net, params, X0, y, 0.01)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.train_step(net, params, X0, y, 0.01)
    el = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 1) for t in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count() or 1
    v = args.steps * Bo / el
    from paper_2203_11014_b200 import configs
    print(json.dumps({
        "impl": "reference", "metric": "DHEN train samples/sec (fwd+bwd)", "value": v, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {configs.DESCR[args.config]}", "global_batch": Bo,
                   "sample_of_batch": configs.BATCH[args.config]},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": int(cores), "kind": "oracle",
                         "sample": f"{args.steps} steps x {Bo} samples of {args.config} (fp64 oracle)"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def relaunch(n: int):
    """--gpus N without a launcher: one process per GPU through torch.distributed.run (rank 0 prints the
    line).  NCCL_DEBUG=INFO goes to stderr so the communicator size (comm nranks) can be checked."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < n:
        raise SystemExit(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default="")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph (launch every kernel from the host)")
    ap.add_argument("--watchdog", action="store_true",
                    help="debug: run the libdhen_wd.so build (bounded mbarrier waits that report and trap)")
    ap.add_argument("--lib", default="", help="debug: load this library build instead (A/B experiments)")
    ap.add_argument("--tuning", default="", help="schedule switches for A/B runs, e.g. sym=1,pair=0 (dhen_tuning)")
    ap.add_argument("--fp", action="store_true",
                    help="NEXT#4 workload: the feature processing layer (configs.FP) in front of the stack, X0 from "
                         "sparse ids and dense features, its backward + sparse SGD after the stack's step")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2203_11014_b200 import binding, configs, flops
    from paper_2203_11014_b200 import build as _build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0 and not os.path.exists(binding.LIB_PATH):
        _build.build()
    if args.watchdog or args.lib:
        binding.load(args.lib or binding.WD_LIB_PATH)
    if world > 1:
        dist.barrier()

    cfg = configs.make(args.config, args.batch or None)
    B = cfg.batch_max_local
    nid = None
    if world > 1:
        obj = [binding.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    model = binding.DHEN(cfg, rank=rank, world=world, nccl_id=nid)
    if args.tuning:
        model.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tuning.split(","))})
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    X0 = synth.make_x0(synth.SEED_BASE + 100 + rank, B, cfg.m0, cfg.d, bf16=(cfg.dtype == "bf16"))
    y = synth.make_labels(synth.SEED_BASE + 100 + rank, B)
    x0 = torch.tensor(X0, device="cuda").to(tdt).contiguous()
    lab = torch.tensor(y, device="cuda")
    fp = None
    if args.fp:   # X0 comes from the feature processing layer; its dX0 drives the sparse SGD
        ntab, R, ndense, hidden, ndtok, mbag = configs.FP[args.config]
        assert ntab + ndtok == cfg.m0
        ids, offs, dense = synth.make_fp_batch(synth.SEED_BASE + 200 + rank, B, [R] * ntab, ndense, mbag,
                                               bf16=(cfg.dtype == "bf16"))
        fp = binding.FeatureProcessing([R] * ntab, ndense, hidden, ndtok, cfg.d, dtype=cfg.dtype, max_batch=B,
                                       max_nnz=len(ids), seed=synth.SEED_BASE + 300)
        t_ids, t_offs = torch.tensor(ids, device="cuda"), torch.tensor(offs, device="cuda")
        t_dense = torch.tensor(dense, device="cuda").to(tdt).contiguous()
        dx0_buf = torch.empty_like(x0)
    loss = torch.zeros(1, device="cuda")
    Bg = B * world
    lr = 0.01
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    graphed = not args.eager

    def step_fp(ids_, offs_, dense_, lab_):
        fp.forward(ids_, offs_, dense_, x0)
        if graphed:
            model.train_step_graphed(x0, lab_, lr, B_global=Bg, loss=loss, dx0=dx0_buf)
        else:
            model.train_step(x0, lab_, lr, B_global=Bg, loss=loss, dx0=dx0_buf)
        fp.backward_sgd(dx0_buf, lr)

    def step():
        if fp is not None:
            step_fp(t_ids, t_offs, t_dense, lab)
        elif graphed:
            model.train_step_graphed(x0, lab, lr, B_global=Bg, loss=loss)
        else:
            model.train_step(x0, lab, lr, B_global=Bg, loss=loss)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device time, L2 flushed before each step)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = model.launches()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(st)
            step()
            ev[k][1].record(st)
        torch.cuda.synchronize()
    launches = model.launches() - l0 - 0
    if world > 1:
        dist.barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([dev_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    value = Bg * args.steps / (dev_ms / 1e3)
    loss_val = float(loss.item())

    # ---------------- e2e: public API with pinned host buffers, copies inside the timed region.  Every step
    # copies its inputs host->device (pinned, on a copy stream, double-buffered: step k+1's upload overlaps
    # step k's compute, as a training input pipeline does), moves them into the step's input buffers and
    # reads the loss back to the host.  The first upload is inside the timed region too.
    if fp is not None:   # the step's host inputs are the ids, offsets and dense features (X0 is computed)
        X0 = dense
    hx = [torch.tensor(X0).to(tdt).pin_memory() for _ in range(2)]
    if fp is not None:
        hids = [torch.tensor(ids).pin_memory() for _ in range(2)]
        hoffs = [torch.tensor(offs).pin_memory() for _ in range(2)]
        stage_i = [torch.empty_like(t_ids) for _ in range(2)]
        stage_o = [torch.empty_like(t_offs) for _ in range(2)]
        di, do = torch.empty_like(t_ids), torch.empty_like(t_offs)
    hy = [torch.tensor(y).pin_memory() for _ in range(2)]
    hl = torch.zeros(1).pin_memory()
    stage_x = [torch.empty_like(t_dense if fp is not None else x0) for _ in range(2)]
    stage_y = [torch.empty_like(lab) for _ in range(2)]
    dx = torch.empty_like(t_dense if fp is not None else x0)
    dy = torch.empty_like(lab)
    cp = torch.cuda.Stream()
    up_done = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dx.copy_(hx[0])
    dy.copy_(hy[0])
    if fp is not None:
        di.copy_(hids[0])
        do.copy_(hoffs[0])

    def e2e_step():
        if fp is not None:
            step_fp(di, do, dx, dy)
        elif graphed:
            model.train_step_graphed(dx, dy, lr, B_global=Bg, loss=loss)
        else:
            model.train_step(dx, dy, lr, B_global=Bg, loss=loss)

    for _ in range(2):   # capture the graph for these buffers outside the timed region
        e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    def upload(k):
        s = k % 2
        with torch.cuda.stream(cp):
            if k >= 2:
                cp.wait_event(used[s])   # the step that read this staging buffer has moved it on
            stage_x[s].copy_(hx[s], non_blocking=True)
            stage_y[s].copy_(hy[s], non_blocking=True)
            if fp is not None:
                stage_i[s].copy_(hids[s], non_blocking=True)
                stage_o[s].copy_(hoffs[s], non_blocking=True)
            up_done[s].record(cp)

    if fp is None:
        # the C ABI's host-buffer entry (dhen_train_step_host): the library uploads each step's pinned host
        # inputs on its own copy stream (two staging slots: step k+1's upload overlaps step k), moves them into
        # the step's input buffers, replays the step graph and copies the loss to a pinned host scalar
        hls = [torch.zeros(1).pin_memory() for _ in range(2)]
        for k in range(2):   # first calls: device buffers and the step graph on them, outside the timed region
            model.train_step_host(hx[k], hy[k], lr, B_global=Bg, loss_host=hls[k], sync=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for k in range(args.steps):
            model.train_step_host(hx[k % 2], hy[k % 2], lr, B_global=Bg, loss_host=hls[k % 2], sync=False)
        e1.record(st)
        torch.cuda.synchronize()
    else:
        e0.record(st)
        cp.wait_event(e0)
        upload(0)
        for k in range(args.steps):
            s = k % 2
            if k + 1 < args.steps:
                upload(k + 1)
            st.wait_event(up_done[s])
            dx.copy_(stage_x[s], non_blocking=True)
            dy.copy_(stage_y[s], non_blocking=True)
            di.copy_(stage_i[s], non_blocking=True)
            do.copy_(stage_o[s], non_blocking=True)
            used[s].record(st)
            e2e_step()
            hl.copy_(loss, non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e = {"value": Bg * args.steps / (e2e_ms / 1e3), "unit": "samples/s",
           "h2d_bytes_per_step": int(hx[0].numel() * hx[0].element_size() + hy[0].numel() * 4 +
                                     (hids[0].numel() * 4 + hoffs[0].numel() * 4 if fp is not None else 0)),
           "d2h_bytes_per_step": 4,
           "pipeline": ("C ABI dhen_train_step_host: " if fp is None else "torch copies around the device-pointer calls: ") +
                       "pinned H2D of step k+1 on a copy stream overlaps step k; D2D into the step buffers; loss D2H"}

    # ---------------- feature processing: device time of its forward and backward + SGD alone (CUDA events)
    fp_info = None
    if fp is not None:
        ef = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        f_ms = b_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            ef[0].record(st)
            fp.forward(t_ids, t_offs, t_dense, x0)
            ef[1].record(st)
            flush.zero_()
            ef[2].record(st)
            fp.backward_sgd(dx0_buf, 0.0)
            ef[3].record(st)
            torch.cuda.synchronize()
            f_ms += ef[0].elapsed_time(ef[1])
            b_ms += ef[2].elapsed_time(ef[3])
        f_ms /= args.steps
        b_ms /= args.steps
        nnz = len(ids)
        es_ = 2 if cfg.dtype == "bf16" else 4
        gather = nnz * cfg.d * 4 + B * ntab * cfg.d * es_ + nnz * 4 + (B * ntab + 1) * 4   # rows, pooled tokens, ids, offsets
        fp_info = {"tables": ntab, "rows_per_table": R, "dense_features": ndense, "hidden": list(hidden),
                   "dense_tokens": ndtok, "mean_bag": mbag, "ids_per_step": nnz,
                   "table_bytes": ntab * R * cfg.d * 4, "fwd_ms": f_ms, "bwd_sgd_ms": b_ms,
                   "share_of_step": (f_ms + b_ms) / (dev_ms / args.steps),
                   "gather_roofline": {"bound": "hbm", "algorithmic_bytes": gather,
                                       "note": "forward incl. the bottom MLP; bytes = looked-up fp32 rows + pooled "
                                               "tokens + ids + offsets",
                                       "achieved_gbs": gather / f_ms / 1e6}}

    # ---------------- profiled pass: per-op device time (roofline of the dominant op)
    model.profile(True)
    for _ in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    ops = model.profile_read()
    model.profile(False)
    tot_ms = sum(o["ms"] for o in ops)
    top = max(ops, key=lambda o: o["ms"])
    pk = peaks()
    per_launch_ms = top["ms"] / top["launches"]
    ai = top["flops"] / max(top["bytes"], 1.0)
    ridge = pk["tc_sus"] * 1e12 / (pk["hbm"] * 1e9)
    is_gemm = top["flops"] > 0 and not top["name"].startswith(("conv", "head", "layer", "attn.soft"))
    tc_path = top.get("tc_launches", 0) > 0
    if is_gemm and ai >= ridge and tc_path:
        bound, unit, achieved, peak = "tensor", "TFLOP/s", top["flops"] / top["ms"] / 1e9, pk["tc_sus"]
    elif is_gemm and not tc_path:
        # exact-FP32 SIMT FMA path: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz
        bound, unit, achieved, peak = "alu", "TFLOP/s", top["flops"] / top["ms"] / 1e9, 148 * 128 * 2 * 1.965e-3
    else:
        bound, unit, achieved, peak = "hbm", "GB/s", top["bytes"] / top["ms"] / 1e6, pk["hbm"]
    # traffic: DRAM bytes per launch of this op's kernel from the committed ncu --set full capture
    # (profiles/ncu_traffic.json, written by tools/ncu_summary.py traffic), when one exists for this op
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        ent = json.load(open(tp)).get(args.config, {}).get(top["name"])
        if ent:
            traffic, traffic_src = ent["traffic_bytes_per_launch"], ent["summary"]
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
            "algorithmic_flops_per_launch": top["flops"] / top["launches"],
            "kernel": top["name"], "share_of_step": top["ms"] / tot_ms,
            "per_launch_ms": per_launch_ms, "launches_per_step": top["launches"] / args.steps,
            "peak_source": pk["src"] + (" sustained bf16" if bound == "tensor" else "")}
    if args.profile_json and rank == 0:
        json.dump({"ops": ops, "steps": args.steps}, open(args.profile_json, "w"), indent=1)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    tf = flops.train_flops_per_sample(cfg)
    es = 2 if cfg.dtype == "bf16" else 4
    step_bytes = sum((3 * mi + 2 * mo) * cfg.d * es for mi, mo in cfg.dims())
    out = {
        "metric": "DHEN train samples/sec (fwd+bwd)", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": f"{args.config}{'+FP' if fp is not None else ''}: {configs.DESCR[args.config]}"
                               f"{' behind the feature processing layer (NEXT#4)' if fp is not None else ''}",
                   "global_batch": Bg, "batch_per_gpu": B,
                   "m0": cfg.m0, "d": cfg.d, "layers": len(cfg.layers),
                   "parallelism": f"fsdp{world}" if world > 1 else "single",
                   **({"tuning": args.tuning} if args.tuning else {}),
                   "l2": "flushed (256 MiB write) before every timed step"},
        "mfu": {"train_flops_per_sample": tf, "vs_burst": value * tf / (world * pk["tc"] * 1e12),
                "vs_sustained": value * tf / (world * pk["tc_sus"] * 1e12)},
        # whole-step rooflines: MFU above; HBM = the step's algorithmic bytes -- per layer X_n read
        # and Y written (forward), X_n and dY read and dX_n written (backward): (3 m_in + 2 m_out) d elements / sample
        "step_hbm": {"alg_bytes_per_sample": step_bytes,
                     "frac": value * step_bytes / (world * pk["hbm"] * 1e9), "peak_gbs": pk["hbm"]},
        "loss": loss_val,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "cuda_graph": graphed and world == 1,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
        "roofline": roof,
        **({"fp": fp_info} if fp_info else {}),
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
