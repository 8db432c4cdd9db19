#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1500 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
echo done
