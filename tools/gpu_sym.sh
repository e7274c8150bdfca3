#!/bin/bash
# A/B of the dot-backward symmetrisation kernel (DHEN_SYM) on C2 / C4 + the dot parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_fusions.py -k symmetris -m gpu -x -q > gpurun_out/sym_pytest.log 2>&1; tail -n 2 gpurun_out/sym_pytest.log
for c in C2 C4; do for v in 0 1 2 0 1 2; do
  env DHEN_SYM=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 --profile-json gpurun_out/sym_${c}_$v.json > gpurun_out/sym_$c.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/sym_$c.json').read().strip().splitlines()[-1]); p=json.load(open('gpurun_out/sym_${c}_$v.json'))
s=[o for o in p['ops'] if o['name']=='dot.sym'][0]; st=p['steps']
print('$c SYM=$v', round(j['value']), round(j['ms_per_step'],4), 'dot.sym ms/step', round(s['ms']/st,4), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done; done
