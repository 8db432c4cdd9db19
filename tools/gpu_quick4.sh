#!/bin/bash
# quick config-4 check: parity subset + one timed call + t=16 K1 profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/q4_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/q4_parity.log
timeout 600 python tools/run_config.py 4 --calls 1 --no-check 2>&1 | tail -c 330 > gpurun_out/q4_c4.log
HT_K1PROF=1 HT_K1PROF_T=0 timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check 2>&1 | grep "K1 cycles per step\|sub-phase" > gpurun_out/q4_prof.log
HT_K1PROF=1 HT_K1PROF_T=16 timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check 2>&1 | grep "K1 cycles per step\|sub-phase" >> gpurun_out/q4_prof.log
