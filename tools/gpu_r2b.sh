#!/bin/bash
# warp-row RQ: unit check + cycles, K1 phase profiles old vs new at r = 64, 128, parity suite
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/rqw_test tools/rqw_test.cu && timeout 120 ./tools/rqw_test > gpurun_out/r2b_rqw_test.log 2>&1
echo "rqw_test rc=$?" >> gpurun_out/r2b_rqw_test.log
for a in "4096 64 32" "4096 128 32"; do
  for lib in new old; do
    L=""; [ $lib = old ] && L="--lib=tools/libht_old.so"
    echo "== $a $lib" >> gpurun_out/r2b_k1prof.log
    HT_K1PROF=1 timeout 600 python tools/k1prof.py $a $L >> gpurun_out/r2b_k1prof.log 2>&1
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
