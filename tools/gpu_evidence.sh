#!/bin/bash
# Round evidence: bench lines (all configs), per-op profiles, C2 ncu launch list, ncu --set full of the
# dominant kernel of each config.  Outputs in gpurun_out/ev_*; summarise with tools/ncu_summary.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
nproc > gpurun_out/ev_host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/ev_host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv >> gpurun_out/ev_host.txt
for c in C2 C3 C4 C5 C1; do
  timeout 600 python bench.py --config $c --profile-json gpurun_out/ev_prof_$c.json > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
  tail -c 200 gpurun_out/ev_bench_$c.json; echo
done
timeout 600 python bench.py --impl reference --config C2 --steps 3 --warmup 3 > gpurun_out/ev_ref_C2.json 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ev_launches_C2.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
echo "launch list rc=$?"
# dominant kernels (skip the warm-up launches, capture one)
cap() {  # config regex skip tag
  timeout 300 python bench.py --config $1 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ev_plain_$4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 \
    -o gpurun_out/ev_ncu_$4 -f python bench.py --config $1 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ev_ncu_$4.log 2>&1
  echo "ncu $4 rc=$?"
}
cap C2 "gemm_tc_kernel<.int.128, .int.4, .int.12" 6 c2_dcn_dT
cap C5 "gemm_tc_kernel<.int.256, .int.3, .int.12" 20 c5_dcn_dT
cap C3 "attn_bwd_kernel" 8 c3_attn_bwd
cap C4 "attn_bwd_kernel" 16 c4_attn_bwd
