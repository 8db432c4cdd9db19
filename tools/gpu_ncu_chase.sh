#!/bin/bash
# one chase_kernel launch (mid reduction) under ncu --set full with source counters -- dev helper
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python tools/k1prof.py 4096 16 32 > gpurun_out/ncu_chase_pre.log 2>&1 || exit 1
HT_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:chase_kernel --launch-skip 40 --launch-count 1 \
  -f -o gpurun_out/prof_chase_now python tools/k1prof.py 4096 16 32 > gpurun_out/ncu_chase.log 2>&1
echo done
