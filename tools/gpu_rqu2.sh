#!/bin/bash
mkdir -p gpurun_out
HT_K1PROF=1 timeout 300 python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/rqu2_k1prof_on.log 2>&1
