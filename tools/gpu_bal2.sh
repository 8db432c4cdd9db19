#!/bin/bash
mkdir -p gpurun_out
for V in "HT_HELPER_BAL=0" "HT_HELPER_BAL=1" "HT_HELPER_BAL=1 HT_HELPER_F=8" "HT_HELPER_BAL=1 HT_HELPER_F=2.5"; do
  echo "== $V" >> gpurun_out/bal2.log
  env $V timeout 600 python tools/run_config.py 4 --calls 2 --no-check 2>&1 | tail -c 230 >> gpurun_out/bal2.log
  echo >> gpurun_out/bal2.log
done
