"""Per-op gap to its own roofline floor from a bench --profile-json dump:
floor = max(flops / bf16 sustained peak, algorithmic bytes / HBM peak).  Usage: gap_table.py prof.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
TF = float(pk.get("bf16_tflops_sustained", 1359.5)) * 1e12
BW = float(pk.get("hbm_gbs", 6547.8)) * 1e9
j = json.load(open(sys.argv[1]))
s = j["steps"]
rows = []
for o in j["ops"]:
    t = o["ms"] / s
    fl = max(o["flops"] / TF, o["bytes"] / BW) * 1e3 / s
    rows.append((t - fl, o["name"], t, fl))
rows.sort(reverse=True)
T = sum(r[2] for r in rows)
F = sum(r[3] for r in rows)
print(f"sum op time {T:.3f} ms/step, sum floors {F:.3f} ms/step ({100 * F / T:.0f}%)")
for g, n, t, fl in rows[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{n:20s} {t:8.3f} ms  floor {fl:8.3f}  gap {g:8.3f}  ({100 * fl / t:4.0f}%)")
