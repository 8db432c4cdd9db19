#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/rep.log
for c in 2 3 4; do
  for late in 0 1; do
    HT_QZ_LATE=$late timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/rep_c${c}_$late.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/rep_c${c}_$late.json')); print('config $c late $late', round(d['ms_per_step'],2), 'ms/step', d['breakdown_ms'])" >> gpurun_out/rep.log
  done
done
