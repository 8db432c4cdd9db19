#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rq_bench tools/rq_bench.cu && ./tools/rq_bench > gpurun_out/rq_bench.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu && ./tools/lat_bench > gpurun_out/lat_bench.log 2>&1
for a in "4096 16 16" "4096 16 8" "4096 16 32" "4096 32 32" "4096 64 32" "2048 32 32 c"; do
  echo "== $a" >> gpurun_out/k1prof.log
  HT_K1PROF=1 timeout 300 python tools/k1prof.py $a >> gpurun_out/k1prof.log 2>&1
done
timeout 300 python tools/k1prof.py 4096 16 16 > gpurun_out/plain_k1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chase -s 300 -c 1 -o gpurun_out/prof_chase_c2 python tools/k1prof.py 4096 16 16 > gpurun_out/ncu_chase.log 2>&1
echo done
