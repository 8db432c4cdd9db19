#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/r3i_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3i_pytest.log
for w in 1 0; do
  HT_WY=$w timeout 900 python tools/run_config.py 4 --calls 2 > gpurun_out/r3i_c4_wy$w.json 2>&1
done
HT_WY=1 timeout 1500 python tools/run_config.py 5 --calls 1 > gpurun_out/r3i_c5_wy1.json 2>&1
