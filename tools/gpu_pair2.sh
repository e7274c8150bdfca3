cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
DHEN_PAIR=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
for pr in 0 1; do
  echo "== DHEN_PAIR=$pr"
  DHEN_PAIR=$pr timeout 120 python tools/gemm_bench.py --cfg C4 --only wgrad 2>&1 | grep -v Warn
  DHEN_PAIR=$pr timeout 120 python tools/gemm_bench.py --cfg C2 --only wgrad 2>&1 | grep -v Warn
done
