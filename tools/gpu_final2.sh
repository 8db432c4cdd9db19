#!/bin/bash
# final evidence: GPU suite, bench lines for configs 4 (default), 2, 3, 5, reference arm
mkdir -p gpurun_out
HT_PARITY_LOG=gpurun_out/f2_parity.jsonl timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f2_pytest.log
timeout 1200 python bench.py > gpurun_out/f2_bench_c4.json 2> gpurun_out/f2_bench_c4.err
timeout 900 python bench.py --config 2 > gpurun_out/f2_bench_c2.json 2> gpurun_out/f2_bench_c2.err
timeout 1200 python bench.py --config 3 --steps 2 > gpurun_out/f2_bench_c3.json 2> gpurun_out/f2_bench_c3.err
timeout 2400 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/f2_bench_c5.json 2> gpurun_out/f2_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f2_bench_ref.json 2> gpurun_out/f2_bench_ref.err
