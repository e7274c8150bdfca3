cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for args in "128 128 300 1" "100 128 300 1" "128 256 200 1" "37 256 50 1"; do
  echo "== $args"; CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_attn.py $args 2>&1 | tail -2
done
timeout 300 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/pytest_attn.log 2>&1; echo "attn rc=$?"; tail -3 gpurun_out/pytest_attn.log
