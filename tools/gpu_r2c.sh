#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/rqw_test > gpurun_out/r2c_rqw_test.log 2>&1
echo "rqw_test rc=$?" >> gpurun_out/r2c_rqw_test.log
for a in "4096 64 32" "4096 128 32"; do
  echo "== $a new" >> gpurun_out/r2c_k1prof.log
  HT_K1PROF=1 timeout 600 python tools/k1prof.py $a >> gpurun_out/r2c_k1prof.log 2>&1
done
