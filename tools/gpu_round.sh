#!/bin/bash
# One GPU round trip: every -m gpu test (errors printed), smoke, then per-op A/B arms (tools/gpu_ab_ops.sh).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rt_build.log 2>&1 || { tail gpurun_out/rt_build.log; exit 1; }
if [ -n "$KEXPR" ]; then
  timeout ${PYT:-1500} python -m pytest tests -m gpu -q -s -k "$KEXPR" > gpurun_out/rt_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rt_pytest.log
else
  timeout ${PYT:-1500} python -m pytest tests -m gpu -q -s > gpurun_out/rt_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rt_pytest.log
fi
tail -n 12 gpurun_out/rt_pytest.log | grep -E "passed|failed|FAILED|rc="
grep -E "^PARITY|^LN offset|^bf16 reduce|world [0-9]:|^probe" gpurun_out/rt_pytest.log > gpurun_out/rt_parity.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rt_smoke.log 2>&1; tail -n 1 gpurun_out/rt_smoke.log
[ -n "$ARMS" ] && bash tools/gpu_ab_ops.sh
exit 0
