#!/bin/bash
# Session-5 closing run: driver-equivalent check, launch list and full ncu captures of the chains, config 5 line
mkdir -p gpurun_out
bash tools/gpu_check.sh
cp gpurun_out/bench_c4.json gpurun_out/final5b_bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/final5b_launches_c4.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/final5b_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"chain_kernel" -s 300 -c 3 -f \
    -o gpurun_out/final5b_chain python tools/run_config.py 4 --calls 1 --no-check > gpurun_out/final5b_ncu_full.log 2>&1
timeout 1500 python bench.py --config 5 --steps 1 > gpurun_out/final5b_bench_c5.json 2> gpurun_out/final5b_bench_c5.err
echo done
