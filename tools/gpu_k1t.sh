#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/k1prof.log
for a in "8192 64 32" "4096 16 32"; do
  for tt in 0 1 16 31; do
    echo "== $a t=$tt" >> gpurun_out/k1prof.log
    HT_K1PROF_T=$tt HT_K1PROF=1 timeout 600 python tools/k1prof.py $a 2>&1 | grep "K1 cyc" | head -1 >> gpurun_out/k1prof.log
  done
done
