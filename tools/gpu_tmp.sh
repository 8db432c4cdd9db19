#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/chp.log
for tl in 74; do
  echo "== tile $tl" >> gpurun_out/chp.log
  HT_CHAIN_PROF_TILE=$tl HT_K1PROF=1 HT_K1PROF_T=0 timeout 300 python tools/k1prof.py 4096 16 32 2>&1 | grep -E "right chain," | tail -1 >> gpurun_out/chp.log
done
HTARGS="4096,16,32 8192,64,32 8192,32,32,c" bash tools/gpu_ht.sh
