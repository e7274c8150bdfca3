cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for dbg in 0 1 3; do
  echo "== DHEN_DBG_EPI=$dbg"
  DHEN_DBG_EPI=$dbg timeout 120 python tools/gemm_bench.py --cfg C4 --only attn.ffn 2>&1 | grep -v Warn
  DHEN_DBG_EPI=$dbg timeout 120 python tools/gemm_bench.py --cfg C4 --only dcn.cross 2>&1 | grep -v Warn
done
echo "== epi mask"; timeout 120 python tools/gemm_bench.py --cfg C4 --only ffn2_dgrad --epi 1
echo "== epi resid"; timeout 120 python tools/gemm_bench.py --cfg C4 --only attn.ffn2 --epi 2
echo "== epi cross"; timeout 120 python tools/gemm_bench.py --cfg C4 --only dcn.cross --epi 3
