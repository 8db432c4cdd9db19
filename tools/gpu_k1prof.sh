#!/bin/bash
# K1 per-phase cycle profile (HT_K1PROF) at the config-4 and config-5 shapes (reduced n) and config 2
mkdir -p gpurun_out
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/k1prof_c4n4096.log 2>&1
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 8192 --calls 1 --no-check > gpurun_out/k1prof_c4n8192.log 2>&1
HT_K1PROF=1 timeout 300 python tools/run_config.py 5 --n 4096 --calls 1 --no-check > gpurun_out/k1prof_c5n4096.log 2>&1
HT_K1PROF=1 timeout 300 python tools/run_config.py 2 --calls 1 --no-check > gpurun_out/k1prof_c2.log 2>&1
HT_K1PROF=1 timeout 300 python tools/run_config.py 3 --n 4096 --calls 1 --no-check > gpurun_out/k1prof_c3n4096.log 2>&1
