#!/bin/bash
# Full GPU validation of the tree: build, every -m gpu test (achieved parity errors printed), smoke, and a
# bench line per config (default = C4).  Logs in gpurun_out/val_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/val_build.log 2>&1 || { echo build failed; tail gpurun_out/val_build.log; exit 1; }
timeout ${PYT:-1500} python -m pytest tests -m gpu -q -s ${PYARGS:-} > gpurun_out/val_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/val_pytest.log
tail -n 3 gpurun_out/val_pytest.log
grep -E "^PARITY|^LN offset|worst" gpurun_out/val_pytest.log > gpurun_out/val_parity.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/val_smoke.log
tail -n 2 gpurun_out/val_smoke.log
for c in ${CFGS:-C4 C2 C3 C5}; do
  timeout 600 python bench.py --config $c > gpurun_out/val_bench_$c.json 2> gpurun_out/val_bench_$c.err
  echo "bench $c rc=$? $(tail -c 300 gpurun_out/val_bench_$c.json | head -c 300)"
done
