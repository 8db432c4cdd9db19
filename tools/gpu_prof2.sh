#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/k1prof.log
for a in "4096 16 32" "8192 64 32"; do
  echo "== $a" >> gpurun_out/k1prof.log
  HT_K1PROF=1 timeout 300 python tools/k1prof.py $a >> gpurun_out/k1prof.log 2>&1
done
timeout 300 python tools/k1prof.py 4096 16 32 > gpurun_out/plain_k1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 200 -c 2 -o gpurun_out/prof_chain_c2 python tools/k1prof.py 4096 16 32 > gpurun_out/ncu_chain.log 2>&1
echo done
