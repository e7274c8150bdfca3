cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python tools/gemm_bench.py --cfg C2 --only dot.proj 2>&1 | grep -v Warn
timeout 120 python tools/gemm_bench.py --cfg C4 --only attn.ffn 2>&1 | grep -v Warn
timeout 120 python tools/gemm_bench.py --cfg C4 --only dot.proj 2>&1 | grep -v Warn
