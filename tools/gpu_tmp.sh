#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/b2.txt
for v in 0 1 0; do
  if [ $v = 1 ]; then export HT_NO_GRAPH=1; else unset HT_NO_GRAPH; fi
  timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e 2>>gpurun_out/b2.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nograph=$v', d['ms_per_step'], d['breakdown_ms'])" >> gpurun_out/b2.txt
done
echo done
