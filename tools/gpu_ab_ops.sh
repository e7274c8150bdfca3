#!/bin/bash
# Per-op A/B on one box: each "label:args" arm runs bench.py with --profile-json; tables via tools/prof_table.py.
# usage: ARMS="r1:--lib paper_2203_11014_b200/libdhen_r1.so cur:" CFGS="C2 C4" tools/gpu_ab_ops.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1 || { tail gpurun_out/ab_build.log; exit 1; }
for c in ${CFGS:-C2 C4 C5}; do
  for arm in $ARMS; do
    lab=${arm%%:*}; a=${arm#*:}; a=${a//;/ }
    timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-20} $a --profile-json gpurun_out/ab_${c}_$lab.json > gpurun_out/ab_${c}_$lab.out 2> gpurun_out/ab_${c}_$lab.err
    python - $c $lab <<'PY'
import json, sys
c, lab = sys.argv[1], sys.argv[2]
try:
    j = json.loads(open(f"gpurun_out/ab_{c}_{lab}.out").read().strip().splitlines()[-1])
    print(f"{c} {lab:8s} value {round(j['value'])} ms {j['ms_per_step']:.3f} clk {j['clocks'].get('sm_mhz')} {j['clocks']['reasons']} top {j['roofline']['kernel']} {j['roofline']['frac']:.3f}")
except Exception as e:
    print(c, lab, "FAILED", e, open(f"gpurun_out/ab_{c}_{lab}.err").read()[-1500:])
PY
    python tools/prof_table.py gpurun_out/ab_${c}_$lab.json > gpurun_out/ab_${c}_$lab.txt 2>/dev/null
  done
done
