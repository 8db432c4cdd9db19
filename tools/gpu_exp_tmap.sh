#!/bin/bash
# Session-5 A/B: 4 x 8 lane map for the transposed (left-update) tile loads / stores
mkdir -p gpurun_out
L=gpurun_out/exp_tmap.log
: > $L
cp tools/libht_tmap.so paper_2301_07964_b200/libht_stage2.so
HT_CHAIN_TMAP=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/exp_tmap_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/exp_tmap_suite.log
for c in 4 3; do
  for v in 0 1; do
    echo "== config $c HT_CHAIN_TMAP=$v" >> $L
    HT_CHAIN_TMAP=$v timeout 900 python tools/run_config.py $c --calls 2 >> $L 2>&1
  done
done
if [ -f oracle_cache/cfg4.npz ]; then bash tools/gpu_c4_parity.sh; fi
