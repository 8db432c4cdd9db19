#!/bin/bash
# bench line (driver contract, default config 4), launch list and one full ncu capture of the chase
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/fb_bench.json 2> gpurun_out/fb_bench.err
echo "bench rc=$?" >> gpurun_out/fb_bench.err
timeout 600 python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/fb_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/fb_launches.csv python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/fb_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:chase -s 20 -c 1 -o gpurun_out/fb_chase python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/fb_ncu_full.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 60 -c 2 -o gpurun_out/fb_chain python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/fb_ncu_chain.log 2>&1
