#!/bin/bash
# GPU check of the headline config: gpu tests, C2 bench + per-op profile, launch list, ncu full of one kernel.
# usage: tools/gpu_c2.sh [ncu-kernel-regex] [config]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
K="${1:-gemm_tc_kernel<128, 4, 12}"
C="${2:-C2}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config $C --profile-json gpurun_out/prof_$C.json > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
tail -c 600 gpurun_out/bench_$C.json
timeout 300 python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$C.csv \
   python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_launch.log 2>&1
[ "$K" = "none" ] || timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:$K" -s 6 -c 1 -o gpurun_out/prof_full_$C -f \
   python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_full.log 2>&1
echo done
