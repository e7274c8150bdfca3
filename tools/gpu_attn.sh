cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 240 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/pytest_attn.log 2>&1; echo "attn rc=$?"; tail -30 gpurun_out/pytest_attn.log
