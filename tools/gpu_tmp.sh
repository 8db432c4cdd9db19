#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
rm -f gpurun_out/k1abs.log
HT_K1PROF=1 HT_K1PROF_T=1 timeout 300 python tools/k1prof.py 8192 64 32 2>&1 | tail -3 >> gpurun_out/k1abs.log
cp exp/libht_stage2.so paper_2301_07964_b200/libht_stage2.so
echo "== exp no prefetch r=64" >> gpurun_out/k1abs.log
HT_K1PROF=1 HT_K1PROF_T=1 timeout 300 python tools/k1prof.py 8192 64 32 2>&1 | tail -3 >> gpurun_out/k1abs.log
