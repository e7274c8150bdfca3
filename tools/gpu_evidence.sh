#!/bin/bash
# Round evidence: bench lines (all configs), per-op profiles, C2 ncu launch list, and one ncu --set full
# capture of each config's dominant op (selected by its NVTX range).  Outputs in gpurun_out/ev_*;
# copy into profiles/ with tools/ev_collect.sh.
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
for c in C2 C3 C4 C5; do
  op=$(python -c "import json; print(json.loads(open('gpurun_out/ev_bench_$c.json').read().strip().splitlines()[-1])['roofline']['kernel'])")
  echo "$c dominant op: $op" > gpurun_out/ev_dom_$c.txt
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ev_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$op/" -s 2 -c 1 \
    -o gpurun_out/ev_ncu_$c -f python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ev_ncu_$c.log 2>&1
  echo "ncu $c $op rc=$?"
done
