cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for s in tokmix.wgrad dcn.wgrad tokmix.fwd; do
  timeout 120 python tools/gemm_bench.py --cfg C2 --only $s --iters 3 > gpurun_out/plain_$s.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemm_tc_kernel" -s 1 -c 1 -o gpurun_out/ncu_c2_$s -f \
     python tools/gemm_bench.py --cfg C2 --only $s --iters 1 > gpurun_out/ncu_c2_$s.log 2>&1
  echo "$s rc=$?"; cat gpurun_out/plain_$s.log | grep -v Warn
done
