#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/chp.log
for tl in 74 100; do
  echo "== WY tile $tl" >> gpurun_out/chp.log
  HT_CHAIN_PROF_TILE=$tl HT_K1PROF=1 HT_K1PROF_T=0 timeout 300 python tools/k1prof.py 4096 16 32 2>&1 | grep -E "right chain," | tail -1 >> gpurun_out/chp.log
done
