cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:attn_(fwd|bwd)_kernel" -s 8 -c 2 -o gpurun_out/ncu_c3_attn -f \
   python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_c3_attn.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_c3_attn.log
