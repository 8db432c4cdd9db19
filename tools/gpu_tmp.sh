#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"accum|merge" -c 8 --csv --log-file gpurun_out/km.csv python tools/k1prof.py 4096 16 32 > /dev/null 2>&1
HTARGS="4096,16,32" bash tools/gpu_ht.sh
