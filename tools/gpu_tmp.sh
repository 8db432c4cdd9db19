#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/ht.log
for kb in 200 224; do
 for a in "8192 64 32" "8192 32 16 c" "4096 16 32"; do
  echo "== $a kb=$kb" >> gpurun_out/ht.log
  HT_CHASE_SMEM_KB=$kb timeout 300 python tools/k1prof.py $a 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
 done
done
