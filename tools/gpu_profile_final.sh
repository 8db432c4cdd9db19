#!/bin/bash
# launch list of the default bench command + one full ncu capture of the chase and chain kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/k1prof.py 4096 16 32 > gpurun_out/plain_k1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"chase_kernel|chain_kernel" -s 300 -c 4 \
    -o gpurun_out/prof_final_c2 python tools/k1prof.py 4096 16 32 > gpurun_out/ncu_full.log 2>&1
echo done
