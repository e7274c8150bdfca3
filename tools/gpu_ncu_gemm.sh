# ncu --set full of one gemm_bench shape.  usage: tools/gpu_ncu_gemm.sh <cfg> <only> <tag> [extra gemm_bench args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python tools/gemm_bench.py --cfg $1 --only $2 --iters 3 $4 > gpurun_out/plain_$3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemm_tc_kernel" -s 1 -c 1 -o gpurun_out/ncu_$3 -f \
   python tools/gemm_bench.py --cfg $1 --only $2 --iters 1 $4 > gpurun_out/ncu_$3.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_$3.log
