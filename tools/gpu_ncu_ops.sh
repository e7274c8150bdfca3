#!/bin/bash
# ncu --set full of selected ops (NVTX range "<op>/") at one config: raw metrics CSV + gzipped source-page CSV.
# usage: CFG=C4 OPS="attn.out_ln1 tokmix.fwd_ln" [TUNING="k=v,k=v"] tools/gpu_ncu_ops.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
CFG=${CFG:-C4}
TU=""; [ -n "$TUNING" ] && TU="--tuning $TUNING"
ECMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --eager $TU"
timeout 600 $ECMD > gpurun_out/no_plain_$CFG.log 2>&1 || { echo "eager plain run failed"; tail gpurun_out/no_plain_$CFG.log; exit 1; }
for op in $OPS; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$op/" -s ${SKIP:-2} -c 1 \
    -o /tmp/no_$op -f $ECMD > gpurun_out/no_${CFG}_$op.log 2>&1
  echo "ncu $CFG $op rc=$?"
  ncu -i /tmp/no_$op.ncu-rep --page raw --csv > gpurun_out/no_raw_${CFG}_$op.csv 2>/dev/null
  ncu -i /tmp/no_$op.ncu-rep --page source --csv --print-source cuda > gpurun_out/no_src_${CFG}_$op.csv 2>/dev/null
  ncu -i /tmp/no_$op.ncu-rep --page source --csv --print-source sass > gpurun_out/no_sass_${CFG}_$op.csv 2>/dev/null
  gzip -f gpurun_out/no_src_${CFG}_$op.csv gpurun_out/no_sass_${CFG}_$op.csv
  rm -f /tmp/no_$op.ncu-rep
done
du -sh gpurun_out
