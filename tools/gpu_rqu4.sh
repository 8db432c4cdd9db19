#!/bin/bash
mkdir -p gpurun_out
for M in 2 1; do
HT_RQU=$M HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu4_k1prof_m$M.log 2>&1
done
