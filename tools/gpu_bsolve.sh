#!/bin/bash
mkdir -p gpurun_out
for m in 64 33 16; do ./tools/rqu_micro $m 200 2; done > gpurun_out/bsolve_micro.log 2>&1
for m in 128 97; do ./tools/rqu_micro128 $m 50 2; done >> gpurun_out/bsolve_micro.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rqu.py -x -q > gpurun_out/bsolve_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/bsolve_parity.log
timeout 600 python tools/run_config.py 4 --calls 2 --no-check 2>&1 | tail -c 230 > gpurun_out/bsolve_c4.log
HT_K1PROF=1 HT_K1PROF_T=16 timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check 2>&1 | grep "K1 cycles per step\|sub-phase" | head -2 >> gpurun_out/bsolve_c4.log
timeout 900 python tools/run_config.py 5 --n 16384 --calls 1 --no-check 2>&1 | tail -c 230 > gpurun_out/bsolve_c5.log
