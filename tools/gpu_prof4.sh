#!/bin/bash
mkdir -p gpurun_out
HT_K1PROF=1 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/prof4_full.log 2>&1
HT_K1PROF=1 HT_K1PROF_T=0 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/prof4_full_t0.log 2>&1
HT_K1PROF=1 HT_K1PROF_T=31 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/prof4_full_t31.log 2>&1
