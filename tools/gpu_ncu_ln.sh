cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --eager --batch 2048 > gpurun_out/plain_ln.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_tc_kernel<.int.256, .int.3, .int.20" -s 4 -c 1 -o gpurun_out/ncu_ln -f \
   python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --eager --batch 2048 > gpurun_out/ncu_ln.log 2>&1
echo "ncu rc=$?"
