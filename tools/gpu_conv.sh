cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --eager --batch 2048 > gpurun_out/plain_conv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:conv_db_k" -s 6 -c 3 -o gpurun_out/ncu_conv -f \
   python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --eager --batch 2048 > gpurun_out/ncu_conv.log 2>&1
echo "ncu rc=$?"
