#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 300 python tools/k1prof.py 8192 64 32 > /dev/null 2>&1 || exit 1
HT_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chase_kernel|chain_kernel" --launch-skip 120 --launch-count 3 \
  -f -o gpurun_out/prof_r64 python tools/k1prof.py 8192 64 32 > gpurun_out/ncu_r64.log 2>&1
