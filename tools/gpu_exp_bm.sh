#!/bin/bash
# Session-5 A/B: chain tiles of 64 rows (tools/libht_bm64.so: -DHT_CHAIN_BM=64) vs 32
mkdir -p gpurun_out
L=gpurun_out/exp_bm.log
: > $L
for c in 4 3 2; do
  echo "== config $c BM=64" >> $L
  timeout 900 python tools/run_config.py $c --lib tools/libht_bm64.so --calls 2 >> $L 2>&1
done
echo "== config 5 BM=64" >> $L
timeout 1500 python tools/run_config.py 5 --lib tools/libht_bm64.so --calls 1 >> $L 2>&1
cp tools/libht_bm64.so paper_2301_07964_b200/libht_stage2.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/exp_bm_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/exp_bm_suite.log
