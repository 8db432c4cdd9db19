#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/k1prof.log
for a in "4096 16 32" "8192 64 32"; do
  for h in "" "HT_NO_HELPERS=1"; do
    echo "== $a $h" >> gpurun_out/k1prof.log
    env $h HT_K1PROF=1 timeout 600 python tools/k1prof.py $a >> gpurun_out/k1prof.log 2>&1
  done
done
