#!/bin/bash
# ncu --set full of one kernel (demangled-name regex) in a short bench run.  usage: tools/gpu_ncu1.sh <regex> <config> <skip> <tag>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config $2 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/plain_$4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:$1" -s $3 -c 1 -o gpurun_out/ncu_$4 -f \
   python bench.py --config $2 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_$4.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$4.log
