#!/bin/bash
# config 4 at full size: per-class device times and the K1 / chain-tile cycle profiles
mkdir -p gpurun_out
HT_K1PROF=1 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/c4prof.log 2>&1
HT_K1PROF=1 HT_CHAIN_PROF_TILE=40 timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/c4prof_t40.log 2>&1
