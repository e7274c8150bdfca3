#!/bin/bash
# Copy a tools/gpu_evidence.sh run from gpurun_out/ into profiles/ (tag r1 = this round)
cd /root/repo
rm -f profiles/ncu_traffic.json profiles/r1_ncu_full_*.txt
for c in C1 C2 C3 C4 C5; do tail -1 gpurun_out/ev_bench_$c.json > profiles/r1_bench_$c.json; python tools/prof_table.py gpurun_out/ev_prof_$c.json > profiles/r1_ops_$c.txt; done
tail -1 gpurun_out/ev_ref_C2.json > profiles/r1_bench_C2_reference.json
cp gpurun_out/ev_launches_C2.csv profiles/r1_launches_C2.csv; python tools/ncu_summary.py launches profiles/r1_launches_C2.csv > profiles/r1_launches_C2_summary.txt
for c in C2 C3 C4 C5; do
  op=$(cut -d' ' -f4 gpurun_out/ev_dom_$c.txt)
  if [ -f gpurun_out/ev_ncu_$c.ncu-rep ]; then
    (cat gpurun_out/ev_dom_$c.txt; python tools/ncu_summary.py full gpurun_out/ev_ncu_$c.ncu-rep) > profiles/r1_ncu_full_$c.txt
    python tools/ncu_summary.py traffic gpurun_out/ev_ncu_$c.ncu-rep $c $op profiles/r1_ncu_full_$c.txt
  fi
done
cp gpurun_out/ev_host.txt profiles/r1_host.txt
for c in C1 C2 C3 C4 C5; do python -c "
import json; j=json.load(open('profiles/r1_bench_$c.json')); r=j['roofline']
print('$c', round(j['value']), round(j['ms_per_step'],3), 'e2e', round(j['e2e']['value']), 'mfu_sus', round(j['mfu']['vs_sustained'],3), r['kernel'], r['bound'], round(r['frac'],3), 'share', round(r['share_of_step'],3), 'cpu', j.get('cpu_baseline',{}).get('value'), j['clocks'].get('sm_mhz'), j['clocks']['reasons'])"; done
