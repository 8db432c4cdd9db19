#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; }
rm -f gpurun_out/qsweep.log
for c in $CFGS; do for q in $QS; do
  echo "== config $c q $q" >> gpurun_out/qsweep.log
  timeout 600 python bench.py --config $c --q $q --steps 2 --warmup 3 --no-cpu --no-e2e >> gpurun_out/qsweep.log 2>&1
done; done
echo done
