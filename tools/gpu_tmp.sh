#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/ht.log
for v in 1 0; do
  for a in "4096 16 32" "8192 64 32" "8192 32 32 c"; do
    echo "== STAIR_FIRST=$v $a" >> gpurun_out/ht.log
    HT_STAIR_FIRST=$v timeout 300 python tools/k1prof.py $a 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
  done
done
