cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for args in "1 128 200 0" "1 128 200 1" "2 128 100 1"; do
  echo "== $args"; CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_attn.py $args 2>&1 | tail -3
done
timeout 600 python -m pytest tests -m gpu -x -q -k "not 1-128-200" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for c in C3 C4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --profile-json gpurun_out/prof_$c.json > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -c 300 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
