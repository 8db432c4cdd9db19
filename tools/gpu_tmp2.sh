#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/rep.log gpurun_out/pyt.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pyt.log 2>&1; echo "pytest rc $?" >> gpurun_out/pyt.log
for i in 1 2 3 4 5; do
  for c in 2 1; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/rep_c${c}_$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/rep_c${c}_$i.json')); print('config $c run $i', round(d['ms_per_step'],2), 'ms/step', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])" >> gpurun_out/rep.log
  done
done
