#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 300 python tools/k1prof.py 8192 64 32 > gpurun_out/ncu_pre64.log 2>&1 || exit 1
HT_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:chase_kernel --launch-skip 60 --launch-count 1 \
  -f -o gpurun_out/prof_chase64 python tools/k1prof.py 8192 64 32 > gpurun_out/ncu_chase64.log 2>&1
