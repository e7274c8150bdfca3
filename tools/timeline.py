"""Print one step of a per-op trace (DHEN.profile_trace / dhen_debug_profile_trace: op, stream, start, end) as a
timeline, ops sorted by start; gap_us = idle time of that op's stream before it (profile(keep_overlap=True) keeps the side stream).
Usage: timeline.py trace.csv steps"""
import sys

rows = [l.strip().split(",") for l in open(sys.argv[1]) if l.strip()]
steps = int(sys.argv[2])
per = len(rows) // steps
last = sorted(rows[-per:], key=lambda r: float(r[2]))
t00 = float(last[0][2])
busy = {}
prev_end = {}
print(f"{'op':22s} st  start_us   dur_us  gap_us")
for op, st, t0, t1 in last:
    t0, t1 = (float(t0) - t00) * 1e3, (float(t1) - t00) * 1e3
    gap = t0 - prev_end.get(st, t0)
    prev_end[st] = t1
    busy[st] = busy.get(st, 0.0) + (t1 - t0)
    print(f"{op:22s} {st:>2s} {t0:9.1f} {t1 - t0:8.1f} {gap:7.1f}")
span = (max(float(r[3]) for r in last) - t00) * 1e3
print(f"span {span:.1f} us; busy per stream: " + ", ".join(f"{k}: {v:.1f}" for k, v in sorted(busy.items())))
