cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python tools/gemm_bench.py --cfg C4 --only fc2_wgrad 2>&1 | grep -v Warn
timeout 120 python tools/gemm_bench.py --cfg C4 --only fc2_wgrad --iters 3 > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/gemm_bench.py --cfg C4 --only fc2_wgrad --iters 2 2>/dev/null | grep -E "gemm|splitk" | awk -F"\",\"" "{print \$5, \$NF}" | tail -6
