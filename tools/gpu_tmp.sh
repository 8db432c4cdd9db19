#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/lov.log
for c in 2 3; do
  for v in 0 1; do
    echo "== config $c HT_NO_LOVERLAP=$v" >> gpurun_out/lov.log
    if [ $v = 1 ]; then export HT_NO_LOVERLAP=1; else unset HT_NO_LOVERLAP; fi
    timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e 2>>gpurun_out/lov.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])" >> gpurun_out/lov.log 2>&1
  done
done
unset HT_NO_LOVERLAP
echo done
