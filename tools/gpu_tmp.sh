#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/rep.log
for v in 0 1; do
  for c in 2 4; do
    if [ $v = 1 ]; then export HT_NO_UV_SPLIT=1; else unset HT_NO_UV_SPLIT; fi
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/rep_${c}_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/rep_${c}_$v.json')); print('config $c nosplit=$v', round(d['ms_per_step'],2), d['breakdown_ms'])" >> gpurun_out/rep.log
  done
done
