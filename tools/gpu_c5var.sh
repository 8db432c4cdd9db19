#!/bin/bash
mkdir -p gpurun_out
for V in "HT_RQU=0" "HT_RQU=2" "HT_HELPERS=3" "HT_HELPERS=3 HT_RQU=0"; do
  echo "== $V" >> gpurun_out/c5var.log
  env $V timeout 600 python tools/run_config.py 5 --n 16384 --calls 1 --no-check 2>&1 | tail -c 300 >> gpurun_out/c5var.log
  echo >> gpurun_out/c5var.log
done
