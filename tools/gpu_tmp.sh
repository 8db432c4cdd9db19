#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/seq.log
for i in 1 2; do
  for smi in 0 1; do
    if [ $smi = 1 ]; then export HT_NO_SMI=1; else unset HT_NO_SMI; fi
    for c in 1 2; do
      timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c nosmi=$smi', round(d['ms_per_step'],2), round(d['breakdown_ms']['total'],1), d['clocks'].get('samples'))" >> gpurun_out/seq.log
    done
  done
done
