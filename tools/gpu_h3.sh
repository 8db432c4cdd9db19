#!/bin/bash
mkdir -p gpurun_out
for V in "HT_HELPERS=3" "HT_HELPERS=3 HT_QZ_GROUPS=0"; do
  echo "== $V" >> gpurun_out/h3.log
  env $V timeout 600 python tools/run_config.py 4 --calls 1 --no-check 2>&1 | tail -c 300 >> gpurun_out/h3.log
  echo >> gpurun_out/h3.log
done
HT_HELPERS=3 HT_K1PROF=1 HT_K1PROF_T=0 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/h3_prof4_t0.log 2>&1
