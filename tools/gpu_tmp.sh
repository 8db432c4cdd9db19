#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HTARGS="4096,16,32 8192,32,32,c 8192,64,32" bash tools/gpu_ht.sh
echo "== HT_MERGE=2 8192,64,32" >> gpurun_out/ht.log
HT_MERGE=2 timeout 300 python tools/k1prof.py 8192 64 32 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
echo "== HT_MERGE=0 8192,32,32,c" >> gpurun_out/ht.log
HT_MERGE=0 timeout 300 python tools/k1prof.py 8192 32 32 c 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"accum|merge" -c 8 --csv --log-file gpurun_out/km.csv python tools/k1prof.py 4096 16 32 > /dev/null 2>&1
