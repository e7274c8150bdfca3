#!/bin/bash
# Round evidence (outputs gpurun_out/ev_*; copy into profiles/ with tools/ev_collect.sh <tag>):
#  * bench lines of every config (the default C4 first) with per-op profiles, and the reference arm;
#  * the ncu launch list of the default bench command (every launch's device time, cold-cache, serialised);
#  * one `ncu --set full` capture per kernel of interest at C4, each selected by its op's NVTX range
#    (eager step: the NVTX ranges exist only when the host launches), for tensor-pipe / DRAM / stall figures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
nproc > gpurun_out/ev_host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/ev_host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv >> gpurun_out/ev_host.txt
for c in ${CFGS:-C4 C2 C3 C5 C1}; do
  timeout 900 python bench.py --config $c --profile-json gpurun_out/ev_prof_$c.json > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err
  echo "bench $c rc=$? $(tail -c 160 gpurun_out/ev_bench_$c.json)"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_ref_C4.json 2>&1
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/ev_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/ev_launches_C4.csv \
   $CMD > gpurun_out/ev_ncu_launch.log 2>&1
echo "launch list rc=$?"
ECMD="python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
timeout 600 $ECMD > gpurun_out/ev_plain_eager.log 2>&1 || { echo "eager plain run failed"; exit 1; }
for op in ${OPS:-dot.proj_ln dot.proj_dgrad dot.proj_wgrad attn.qkv attn.ffn1 attn.ffn2_ln2 attn.ffn2_dgrad attn.ffn1_wgrad attn.core attn.core_bwd dcn.dT_fused dot.gram_bwd}; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$op/" -s 2 -c 1 \
    -o /tmp/ev_ncu_C4_$op -f $ECMD > gpurun_out/ev_ncu_C4_$op.log 2>&1
  echo "ncu C4 $op rc=$?"
  # keep the raw metrics (small) and a source-level stall table; the report itself stays on the box
  ncu -i /tmp/ev_ncu_C4_$op.ncu-rep --page raw --csv > gpurun_out/ev_raw_C4_$op.csv 2>/dev/null
  ncu -i /tmp/ev_ncu_C4_$op.ncu-rep --page source --csv --print-source cuda > /tmp/src_$op.csv 2>/dev/null && \
    python tools/ncu_summary.py source /tmp/src_$op.csv > gpurun_out/ev_src_C4_$op.txt 2>&1
  rm -f /tmp/ev_ncu_C4_$op.ncu-rep /tmp/src_$op.csv
done
gzip -f gpurun_out/ev_launches_C4.csv 2>/dev/null
du -sh gpurun_out
