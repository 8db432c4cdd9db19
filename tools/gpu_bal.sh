#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_protocol.py -x -q > gpurun_out/bal_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/bal_parity.log
for V in "HT_HELPER_BAL=1" "HT_HELPER_BAL=0" "HT_HELPER_F=3" "HT_HELPER_F=10"; do
  echo "== $V" >> gpurun_out/bal.log
  env $V timeout 600 python tools/run_config.py 4 --calls 1 --no-check 2>&1 | tail -c 330 >> gpurun_out/bal.log
  echo >> gpurun_out/bal.log
done
HT_K1PROF=1 HT_K1PROF_T=0 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/bal_prof4_t0.log 2>&1
