#!/bin/bash
mkdir -p gpurun_out
for a in "4096 64 32" "4096 128 32"; do
  echo "== $a" >> gpurun_out/r2v_k1prof.log
  HT_K1PROF=1 timeout 600 python tools/k1prof.py $a >> gpurun_out/r2v_k1prof.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/r2v_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2v_pytest.log
