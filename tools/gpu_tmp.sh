#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/rep.log
for i in 1 2 3 4 5; do
  for c in 1 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/rep_c${c}_$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/rep_c${c}_$i.json')); print('config $c run $i', round(d['ms_per_step'],2), 'ms/step', round(d['value'],1), d['unit'], 'clocks', d['clocks'])" >> gpurun_out/rep.log
  done
done
