#!/bin/bash
# build, gpu tests, per-op profiled bench of the given configs.  usage: tools/gpu_quick.sh C2 C5 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --profile-json gpurun_out/prof_$c.json > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    j = json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
    print(c, "value", round(j["value"]), "ms", round(j["ms_per_step"], 3), "e2e", round(j["e2e"]["value"]), "clk", j["clocks"].get("sm_mhz"), j["clocks"]["reasons"], "top", j["roofline"]["kernel"], round(j["roofline"]["frac"], 3))
except Exception as e:
    print(c, "FAILED", e); print(open(f"gpurun_out/bench_{c}.err").read()[-2000:])
PY
done
