#!/bin/bash
# Copy a tools/gpu_evidence.sh run from gpurun_out/ into profiles/ with round tag $1 (e.g. r2).
cd /root/repo; T=${1:-r2}
for c in C1 C2 C3 C4 C5; do
  [ -f gpurun_out/ev_bench_$c.json ] || continue
  tail -1 gpurun_out/ev_bench_$c.json > profiles/${T}_bench_$c.json
  python tools/prof_table.py gpurun_out/ev_prof_$c.json > profiles/${T}_ops_$c.txt
done
[ -f gpurun_out/ev_ref_C4.json ] && tail -1 gpurun_out/ev_ref_C4.json > profiles/${T}_bench_C4_reference.json
if [ -f gpurun_out/ev_launches_C4.csv.gz ]; then
  cp gpurun_out/ev_launches_C4.csv.gz profiles/${T}_launches_C4.csv.gz
  gunzip -c profiles/${T}_launches_C4.csv.gz > /tmp/launches.csv
  python tools/ncu_summary.py launches /tmp/launches.csv > profiles/${T}_launches_C4_summary.txt
fi
rm -f profiles/${T}_ncu_C4_*.txt
for f in gpurun_out/ev_raw_C4_*.csv; do
  [ -s "$f" ] || continue
  op=$(basename $f .csv); op=${op#ev_raw_C4_}
  (echo "C4 op $op (ncu --set full --clock-control none, one launch after warm-up, NVTX range $op/)"
   python tools/ncu_summary.py full $f
   [ -f gpurun_out/ev_src_C4_$op.txt ] && { echo "--- source lines with the most warp stall samples"; cat gpurun_out/ev_src_C4_$op.txt; }
  ) > profiles/${T}_ncu_C4_$op.txt
  python tools/ncu_summary.py traffic $f C4 $op profiles/${T}_ncu_C4_$op.txt
done
cp gpurun_out/ev_host.txt profiles/${T}_host.txt 2>/dev/null
