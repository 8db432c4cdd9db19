#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/rep.log
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/rep_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rep_$i.json')); print('run $i', round(d['ms_per_step'],2), 'ms/step', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/rep.log
done
