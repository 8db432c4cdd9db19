#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/rqu5_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/rqu5_parity.log
HT_K1PROF=1 timeout 300 python tools/run_config.py 5 --n 4096 --calls 1 --no-check > gpurun_out/rqu5_k1prof_c5n4096.log 2>&1
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu5_k1prof_c4n4096.log 2>&1
timeout 1200 python tools/run_config.py 5 --calls 1 > gpurun_out/rqu5_c5.json 2>&1
timeout 900 python tools/run_config.py 4 --calls 2 > gpurun_out/rqu5_c4.json 2>&1
