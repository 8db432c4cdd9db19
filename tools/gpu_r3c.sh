#!/bin/bash
mkdir -p gpurun_out
for L in pipe0 pipe2; do
  timeout 900 python tools/run_config.py 4 --calls 2 --lib=tools/libht_$L.so > gpurun_out/r3c_c4_$L.json 2>&1
  timeout 900 python tools/run_config.py 2 --calls 3 --lib=tools/libht_$L.so > gpurun_out/r3c_c2_$L.json 2>&1
  timeout 900 python tools/run_config.py 3 --calls 2 --no-check --lib=tools/libht_$L.so > gpurun_out/r3c_c3_$L.json 2>&1
done
