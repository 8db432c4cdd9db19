#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/rqu3_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/rqu3_parity.log
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu3_k1prof.log 2>&1
timeout 900 python tools/run_config.py 4 --calls 2 > gpurun_out/rqu3_c4.json 2>&1
