#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/k1abs.log
for a in "8192 64 32" "8192 32 32 c" "4096 16 32"; do
  echo "== base $a" >> gpurun_out/k1abs.log
  HT_K1PROF=1 HT_K1PROF_T=1 timeout 300 python tools/k1prof.py $a 2>&1 | grep -E "K1 cycles per step|wall" >> gpurun_out/k1abs.log
done
cp exp/libht_stage2.so paper_2301_07964_b200/libht_stage2.so
for a in "8192 64 32" "8192 32 32 c" "4096 16 32"; do
  echo "== SPR128 $a" >> gpurun_out/k1abs.log
  HT_K1PROF=1 HT_K1PROF_T=1 timeout 300 python tools/k1prof.py $a 2>&1 | grep -E "K1 cycles per step|wall" >> gpurun_out/k1abs.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q >> gpurun_out/k1abs.log 2>&1
