#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for L in "" "--lib=tools/libht_minb2.so"; do
  tag=$( [ -z "$L" ] && echo def || echo minb2 )
  timeout 900 python tools/run_config.py 4 --calls 2 --no-check $L > gpurun_out/r3b_c4_${tag}_$rep.json 2>&1
done
done
timeout 900 python tools/run_config.py 2 --calls 3 --no-check --lib=tools/libht_minb2.so > gpurun_out/r3b_c2_minb2.json 2>&1
timeout 900 python tools/run_config.py 2 --calls 3 --no-check > gpurun_out/r3b_c2_def.json 2>&1
