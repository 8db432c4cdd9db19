#!/bin/bash
# driver-equivalent check: GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "bench rc=$?" >> gpurun_out/bench_c4.err
