"""Summarise ncu outputs for profiles/.
    python tools/ncu_summary.py launches <launches.csv>      -> per-kernel share of device time
    python tools/ncu_summary.py full <report.ncu-rep>        -> key metrics of a --set full capture
    python tools/ncu_summary.py sass <sass-page.csv>         -> warp-stall samples per SASS instruction / region
    python tools/ncu_summary.py traffic <report.ncu-rep> <config> <op> <summary.txt>
        -> add {config: {op: dram bytes per launch, ncu duration}} to profiles/ncu_traffic.json (read by bench.py
           to fill roofline.traffic for that op)"""
import json
import os
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, cold-cache, serialised): {sum(v[0] for v in agg.values())} launches, {tot/1e3:.1f} us total")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t/1e3:10.1f} {100*t/tot:6.1f}%")


def _raw(path):
    """The raw-page CSV of a report (.ncu-rep), or a saved raw CSV (.csv)."""
    if path.endswith(".csv"):
        return open(path).read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout


def full(path):
    out = _raw(path)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_tensor.sum", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "smsp__inst_executed.sum"]
    want += ["lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
    for r in rows[2:]:
        print("---")
        stalls = []
        for h, u, v in zip(hdr, units, r):
            if h in want or (("pipe_tensor" in h or "tmem" in h or "pipe_uma" in h or "tcgen" in h) and "pct" in h):
                print(f"{h} [{u}] = {v}")
            elif h.startswith("smsp__average_warp_latency_issue_stalled_") or \
                    (h.startswith("smsp__warp_issue_stalled_") and h.endswith("per_warp_active.pct")):
                try:
                    stalls.append((float(v.replace(",", "")), h, u))
                except ValueError:
                    pass
        for val, h, u in sorted(stalls, reverse=True)[:8]:
            print(f"stall {h} [{u}] = {val}")


def traffic(path, cfg, op, summary):
    out = _raw(path)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    r = rows[2]
    get = lambda k: r[hdr.index(k)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    nbytes = sum(float(get(k).replace(",", "")) * scale[units[hdr.index(k)]]
                 for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    dur = float(get("gpu__time_duration.sum").replace(",", ""))
    dur_us = dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                    "second": 1e6, "s": 1e6}[units[hdr.index("gpu__time_duration.sum")]]
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    j = json.load(open(p)) if os.path.exists(p) else {}
    j.setdefault(cfg, {})[op] = {"kernel": get("Kernel Name"), "traffic_bytes_per_launch": nbytes,
                                 "ncu_duration_us": dur_us, "summary": summary,
                                 "how": "ncu --set full --clock-control none, one launch after warm-up; "
                                        "dram__bytes_read.sum + dram__bytes_write.sum (writes still dirty in the "
                                        "126 MB L2 when the kernel ends are not counted)"}
    json.dump(j, open(p, "w"), indent=1, sort_keys=True)
    print(f"{cfg} {op}: {nbytes / 1e6:.1f} MB per launch, {dur_us:.1f} us under ncu")


def source(path, top=15):
    """Top source lines by warp-stall samples from `ncu -i rep --page source --csv --print-source cuda`."""
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next((i for i, r in enumerate(rows) if any("Stall" in c or "Sampl" in c for c in r)), None)
    if hi is None:
        print("(no stall-sampling columns found; header:", rows[0][:12] if rows else [], ")")
        return
    hdr = rows[hi]
    samp = [i for i, c in enumerate(hdr) if "Sampl" in c and "All" in c] or \
           [i for i, c in enumerate(hdr) if "Stall" in c or "Sampl" in c]
    src = next((i for i, c in enumerate(hdr) if c.strip().lower() in ("source", "cuda source")), None)
    line = next((i for i, c in enumerate(hdr) if c.strip() in ("#", "Line", "Line Number")), None)
    k = samp[0]
    recs = []
    for r in rows[hi + 1:]:
        try:
            v = float(r[k].replace(",", ""))
        except (ValueError, IndexError):
            continue
        recs.append((v, r[line] if line is not None else "", (r[src] if src is not None else "").strip()[:110]))
    tot = sum(v for v, _, _ in recs) or 1.0
    print(f"column '{hdr[k]}', {int(tot)} samples")
    for v, ln, tx in sorted(recs, reverse=True)[:top]:
        print(f"{100 * v / tot:5.1f}%  line {ln:>5}  {tx}")


def sass(path, top=25, bucket=100):
    """Stall sampling per SASS instruction from `ncu -i rep --page source --csv --print-source sass`: the top
    instructions (with their neighbours' opcodes) and a histogram over 100-instruction regions."""
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next((i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r), None)
    if hi is None:
        print("(no SASS stall-sampling table)")
        return
    hdr = rows[hi]
    iS, iE, iT = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
    data = rows[hi + 1:]
    val = lambda r: float((r[iS] or "0").replace(",", ""))
    tot = sum(val(r) for r in data) or 1.0
    print(f"{int(tot)} warp-stall samples over {len(data)} SASS instructions"
          f"{' (kernel: ' + rows[0][1][:90] + ')' if rows[0] and rows[0][0] == 'Kernel Name' else ''}")
    print("-- top instructions (share of samples, times executed, instruction)")
    for i in sorted(sorted(range(len(data)), key=lambda i: -val(data[i]))[:top]):
        print(f"{i:5d} {100 * val(data[i]) / tot:5.1f}% {data[i][iE]:>10s}  {data[i][iT].strip()[:80]}")
    print(f"-- regions of {bucket} instructions with >= 2 % of the samples")
    for b in range(0, len(data), bucket):
        sh = sum(val(r) for r in data[b:b + bucket]) / tot
        if sh >= 0.02:
            ops = defaultdict(int)
            for r in data[b:b + bucket]:
                t = r[iT].strip().split()
                if t:
                    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
                    ops[op.split(".")[0]] += 1
            top_ops = ",".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
            print(f"{b:5d}-{b + bucket:<5d} {100 * sh:5.1f}%  {top_ops}")


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(*sys.argv[2:6])
    else:
        {"launches": launches, "full": full, "source": source, "sass": sass}[sys.argv[1]](sys.argv[2])
