cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for pr in 0 1; do
  echo "== DHEN_PAIR=$pr"
  DHEN_PAIR=$pr timeout 120 python tools/gemm_bench.py --cfg C2 --only dot.proj 2>&1 | grep -v Warn
  DHEN_PAIR=$pr timeout 120 python tools/gemm_bench.py --cfg C4 --only dot.proj 2>&1 | grep -v Warn
done
for pr in 0 1; do DHEN_PAIR=$pr timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 30 > gpurun_out/pair_$pr.json 2>&1; python -c "
import json; j=json.loads(open('gpurun_out/pair_$pr.json').read().strip().splitlines()[-1]); print('C2 pair=$pr', j['value'], j['ms_per_step'])"; done
