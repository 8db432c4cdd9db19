#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/r2x_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2x_pytest.log
for g in 1 0; do
  HT_QZ_GROUPS=$g timeout 900 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/r2x_c4_g$g.json 2>&1
  HT_QZ_GROUPS=$g timeout 900 python tools/run_config.py 2 --calls 3 --no-check > gpurun_out/r2x_c2_g$g.json 2>&1
done
