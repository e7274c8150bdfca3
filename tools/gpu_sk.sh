cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 nsys --version >/dev/null 2>&1
timeout 120 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/plain_sk.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:splitk|gemm_tc_kernel<64, 6, 0|gemm_tc_kernel<128, 4, 0" --csv --log-file gpurun_out/sk.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --eager > /dev/null 2>&1
echo rc=$?
