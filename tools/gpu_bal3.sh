#!/bin/bash
mkdir -p gpurun_out
for V in "HT_HELPER_BAL=1 HT_HELPER_F=12" "HT_HELPER_BAL=1 HT_HELPER_F=20"; do
  echo "== c4 $V" >> gpurun_out/bal3.log
  env $V timeout 600 python tools/run_config.py 4 --calls 2 --no-check 2>&1 | tail -c 230 >> gpurun_out/bal3.log
  echo >> gpurun_out/bal3.log
done
for V in "HT_HELPER_BAL=0" "HT_HELPER_BAL=1 HT_HELPER_F=8" "HT_HELPER_BAL=1 HT_HELPER_F=16"; do
  echo "== c5n16384 $V" >> gpurun_out/bal3.log
  env $V timeout 600 python tools/run_config.py 5 --n 16384 --calls 1 --no-check 2>&1 | tail -c 230 >> gpurun_out/bal3.log
  echo >> gpurun_out/bal3.log
done
