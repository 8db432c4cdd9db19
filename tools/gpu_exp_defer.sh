#!/bin/bash
# Session-5: far band rows deferred to the apply phase (defer_far, q <= r + 1)
mkdir -p gpurun_out
L=gpurun_out/exp_defer.log
: > $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_protocol.py tests/test_gpu_rqu.py -x -q > gpurun_out/exp_defer_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/exp_defer_suite.log
echo "== config 4 defer (default)" >> $L
timeout 900 python tools/run_config.py 4 --calls 2 >> $L 2>&1
echo "== config 4 defer HT_HELPER_LAG=1" >> $L
HT_HELPER_LAG=1 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
echo "== config 4 defer HT_HELPERS=1" >> $L
HT_HELPERS=1 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
echo "== config 4 defer HT_HELPERS=1 HT_HELPER_LAG=1" >> $L
HT_HELPERS=1 HT_HELPER_LAG=1 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
echo "== config 4 HT_DEFER_FAR=0" >> $L
HT_DEFER_FAR=0 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
echo "== config 3 defer (default)" >> $L
timeout 900 python tools/run_config.py 3 --calls 2 >> $L 2>&1
echo "== config 3 defer HT_HELPERS=1" >> $L
HT_HELPERS=1 timeout 900 python tools/run_config.py 3 --calls 2 --no-check >> $L 2>&1
echo "== config 5 defer (default)" >> $L
timeout 1500 python tools/run_config.py 5 --calls 1 >> $L 2>&1
echo "== config 5 defer HT_HELPERS=1" >> $L
HT_HELPERS=1 timeout 1500 python tools/run_config.py 5 --calls 1 --no-check >> $L 2>&1
