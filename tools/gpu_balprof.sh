#!/bin/bash
mkdir -p gpurun_out
for T in 0 4 8 12 16 20 24 28 31; do
  echo "== t=$T" >> gpurun_out/balprof.log
  HT_K1PROF=1 HT_K1PROF_T=$T timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check 2>&1 | grep "K1 cycles per step" >> gpurun_out/balprof.log
done
