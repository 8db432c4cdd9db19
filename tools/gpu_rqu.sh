#!/bin/bash
# RQ-update chase (rqu.cuh): parity, config-4 timing on/off, K1 phase profile
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/rqu_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/rqu_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/rqu_parity.log
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu_k1prof_on.log 2>&1
HT_RQU=0 HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu_k1prof_off.log 2>&1
timeout 900 python tools/run_config.py 4 --calls 2 > gpurun_out/rqu_c4_on.json 2>&1
