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
timeout 900 python bench.py --config C4 --fp --no-cpu-baseline > gpurun_out/ev_bench_C4fp.json 2> gpurun_out/ev_bench_C4fp.err
echo "bench C4+FP rc=$? $(tail -c 160 gpurun_out/ev_bench_C4fp.json)"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_ref_C4.json 2>&1
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/ev_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/ev_launches_C4.csv \
   $CMD > gpurun_out/ev_ncu_launch.log 2>&1
echo "launch list rc=$?"
ECMD="python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
timeout 600 $ECMD > gpurun_out/ev_plain_eager.log 2>&1 || { echo "eager plain run failed"; exit 1; }
ncu_ops() {   # $1 config, $2 eager bench command, rest: ops (NVTX ranges)
  local c=$1 cmd=$2; shift 2
  for op in "$@"; do
    timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$op/" -s 2 -c 1 \
      -o /tmp/ev_ncu_${c}_$op -f $cmd > gpurun_out/ev_ncu_${c}_$op.log 2>&1
    echo "ncu $c $op rc=$?"
    # keep the raw metrics (small) and the per-SASS-instruction stall table; the report itself stays on the box
    ncu -i /tmp/ev_ncu_${c}_$op.ncu-rep --page raw --csv > gpurun_out/ev_raw_${c}_$op.csv 2>/dev/null
    ncu -i /tmp/ev_ncu_${c}_$op.ncu-rep --page source --csv --print-source sass > /tmp/sass_$op.csv 2>/dev/null && \
      python tools/ncu_summary.py sass /tmp/sass_$op.csv > gpurun_out/ev_src_${c}_$op.txt 2>&1
    rm -f /tmp/ev_ncu_${c}_$op.ncu-rep /tmp/sass_$op.csv
  done
}
ncu_ops C4 "$ECMD" ${OPS:-dot.proj_ln dot.proj_dgrad dot.proj_wgrad attn.qkv attn.ffn1 attn.ffn2_ln2 attn.ffn2_dgrad attn.ffn1_wgrad attn.core attn.core_bwd dcn.bwd_fused dot.gram_bwd attn.out_ln1 tokmix.fwd_ln tokmix.dgrad}
ncu_ops C5 "python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --eager" dcn.bwd_fused dcn.cross
gzip -f gpurun_out/ev_launches_C4.csv 2>/dev/null
du -sh gpurun_out
