#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 300 python tools/k1prof.py 4096 16 32 > /dev/null 2>&1 || exit 1
HT_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel --launch-skip 128 --launch-count 1 \
  -f -o gpurun_out/prof_chainR python tools/k1prof.py 4096 16 32 > gpurun_out/ncu_chainR.log 2>&1
