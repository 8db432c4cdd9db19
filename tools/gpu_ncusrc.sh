#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chase_kernel -s 40 -c 1 -o gpurun_out/chase_src -f python tools/run_config.py 4 --n 4096 --calls 1 --no-check > gpurun_out/ncusrc.log 2>&1
echo "rc=$?" >> gpurun_out/ncusrc.log
