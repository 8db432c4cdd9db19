#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HTARGS="4096,16,32 8192,64,32 8192,32,16,c" bash tools/gpu_ht.sh
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/b2.json 2> gpurun_out/b2.err
