#!/bin/bash
mkdir -p gpurun_out
for W in 1; do
HT_K1PROF=1 HT_K1PROF_T=16 timeout 600 python tools/noqz_prof.py 4 8192 $W 2>&1 | grep "K1 cycles per step\|sub-phase\|withqz" >> gpurun_out/noqz.log
done
