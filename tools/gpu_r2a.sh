#!/bin/bash
# round-2 first GPU call: suite (with full-size parity log), bench config 4 (default), config 5 once
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
HT_PARITY_LOG=gpurun_out/r2a_parity.jsonl timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 900 python bench.py > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err
echo "bench rc=$?" >> gpurun_out/r2a_bench_c4.err
timeout 1200 python tools/run_config.py 5 --calls 1 > gpurun_out/r2a_cfg5.json 2> gpurun_out/r2a_cfg5.err
echo "cfg5 rc=$?" >> gpurun_out/r2a_cfg5.err
