"""Print a per-op table from a bench --profile-json dump."""
import json
import sys

j = json.load(open(sys.argv[1]))
ops = sorted(j["ops"], key=lambda o: -o["ms"])
T = sum(o["ms"] for o in ops)
print(f"total {T / j['steps']:.3f} ms/step (profiled)")
for o in ops:
    print(f"{o['name']:20s} {o['launches']:5d} tc={o['tc_launches']:4d} {o['ms'] / j['steps']:8.3f} ms/step "
          f"{100 * o['ms'] / T:5.1f}%  {o['flops'] / o['ms'] / 1e9:8.1f} TF/s {o['bytes'] / o['ms'] / 1e6:8.1f} GB/s")
