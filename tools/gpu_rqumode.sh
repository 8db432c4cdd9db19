#!/bin/bash
# RQ-update mode / helper balance A/B at config 4 (full size), plus n=8192 traces
mkdir -p gpurun_out
HT_RQU=1 timeout 600 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/ab_rqu1.json 2>&1
HT_HELPER_F=20 timeout 600 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/ab_f20.json 2>&1
HT_HELPER_F=5 timeout 600 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/ab_f5.json 2>&1
HT_RQU=1 HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_rqu1.bin timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check > /dev/null 2>&1
python tools/trace_path.py gpurun_out/tr_rqu1.bin > gpurun_out/trace_rqu1.txt 2>&1
