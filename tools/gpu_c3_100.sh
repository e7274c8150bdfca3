#!/bin/bash
# 100 consecutive default C3 bench runs (the round-1 hang's acceptance check), each under a kill timeout.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c3_build.log 2>&1 || exit 1
${PRE:-true}
ok=0; bad=0
for i in $(seq 1 ${NB:-100}); do
  timeout -s KILL 120 python bench.py --config C3 --no-cpu-baseline > gpurun_out/c3r_last.json 2> gpurun_out/c3r_last.err
  rc=$?
  if [ $rc -eq 0 ]; then ok=$((ok+1)); v=$(python -c "import json;print(round(json.loads(open('gpurun_out/c3r_last.json').read().strip().splitlines()[-1])['value']))"); else bad=$((bad+1)); v=-; cp gpurun_out/c3r_last.err gpurun_out/c3r_fail_$i.err; fi
  echo "run $i rc=$rc samples/s=$v" >> gpurun_out/c3_100.txt
done
echo "C3 bench x ${NB:-100}: ok=$ok failed=$bad" | tee -a gpurun_out/c3_100.txt
