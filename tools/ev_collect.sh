#!/bin/bash
# Copy a tools/gpu_evidence.sh run from gpurun_out/ into profiles/ with round tag $1 (e.g. r2).
cd /root/repo; T=${1:-r2}
for c in C1 C2 C3 C4 C5 C4fp; do
  [ -f gpurun_out/ev_bench_$c.json ] || continue
  tail -1 gpurun_out/ev_bench_$c.json > profiles/${T}_bench_$c.json
  [ -f gpurun_out/ev_prof_$c.json ] && python tools/prof_table.py gpurun_out/ev_prof_$c.json > profiles/${T}_ops_$c.txt
  [ -f gpurun_out/ev_prof_$c.json ] && python tools/gap_table.py gpurun_out/ev_prof_$c.json 40 > profiles/${T}_roofline_gap_$c.txt
done
[ -f gpurun_out/ev_ref_C4.json ] && tail -1 gpurun_out/ev_ref_C4.json > profiles/${T}_bench_C4_reference.json
if [ -f gpurun_out/ev_launches_C4.csv.gz ]; then
  cp gpurun_out/ev_launches_C4.csv.gz profiles/${T}_launches_C4.csv.gz
  gunzip -c profiles/${T}_launches_C4.csv.gz > /tmp/launches.csv
  python tools/ncu_summary.py launches /tmp/launches.csv > profiles/${T}_launches_C4_summary.txt
fi
rm -f profiles/${T}_ncu_C*_*.txt
for f in gpurun_out/ev_raw_C*_*.csv; do
  [ -s "$f" ] || continue
  b=$(basename $f .csv); b=${b#ev_raw_}; c=${b%%_*}; op=${b#*_}
  (echo "$c op $op (ncu --set full --clock-control none, one launch after warm-up, NVTX range $op/)"
   python tools/ncu_summary.py full $f
   [ -f gpurun_out/ev_src_${c}_$op.txt ] && { echo "--- warp-stall samples by SASS instruction"; cat gpurun_out/ev_src_${c}_$op.txt; }
  ) > profiles/${T}_ncu_${c}_$op.txt
  python tools/ncu_summary.py traffic $f $c $op profiles/${T}_ncu_${c}_$op.txt
done
cp gpurun_out/ev_host.txt profiles/${T}_host.txt 2>/dev/null
