#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q -k "FAR_SIDE" > gpurun_out/r3a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3a_pytest.log
for f in 0 1; do
  HT_FAR_SIDE=$f timeout 900 python tools/run_config.py 4 --calls 3 --no-check > gpurun_out/r3a_c4_f$f.json 2>&1
  HT_FAR_SIDE=$f timeout 900 python tools/run_config.py 2 --calls 4 --no-check > gpurun_out/r3a_c2_f$f.json 2>&1
  HT_FAR_SIDE=$f timeout 900 python tools/run_config.py 3 --calls 2 --no-check > gpurun_out/r3a_c3_f$f.json 2>&1
done
HT_FAR_SIDE=1 timeout 900 python tools/run_config.py 5 --calls 1 --no-check > gpurun_out/r3a_c5_f1.json 2>&1
