#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/far_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/far_parity.log
HT_K1PROF=1 HT_K1PROF_T=0 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/far_prof4_t0.log 2>&1
timeout 900 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/far_c4.json 2>&1
timeout 900 python tools/run_config.py 3 --calls 2 --no-check > gpurun_out/far_c3.json 2>&1
timeout 900 python tools/run_config.py 2 --calls 3 --no-check > gpurun_out/far_c2.json 2>&1
