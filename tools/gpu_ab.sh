# A/B an env switch on bench lines: tools/gpu_ab.sh VAR "C2 C5" [steps] ["values"]
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for c in $2; do for v in ${4:-0 1 0 1}; do
  env $1=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps ${3:-30} --profile-json gpurun_out/ab_${c}_$v.json > gpurun_out/ab_$c.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/ab_$c.json').read().strip().splitlines()[-1]); print('$c $1=$v', round(j['value']), round(j['ms_per_step'],4), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done; done
