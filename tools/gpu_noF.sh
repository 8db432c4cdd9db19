#!/bin/bash
mkdir -p gpurun_out
for L in paper_2301_07964_b200/libht_stage2.so tools/libht_l2.so; do
echo "== $L" >> gpurun_out/noF.log
HT_K1PROF=1 HT_K1PROF_T=16 timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check --lib $L 2>&1 | grep "K1 cycles per step\|sub-phase" | head -2 >> gpurun_out/noF.log
done
