#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/ht.log
for v in base bz8; do
  if [ $v = bz8 ]; then cp exp8/libht_stage2.so paper_2301_07964_b200/libht_stage2.so; fi
  for a in "4096 16 32" "8192 64 32" "8192 32 32 c"; do
    echo "== $v $a" >> gpurun_out/ht.log
    timeout 300 python tools/k1prof.py $a 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q >> gpurun_out/ht.log 2>&1
