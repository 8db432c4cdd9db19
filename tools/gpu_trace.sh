#!/bin/bash
# chase critical-path traces (HT_LAG_CHECK stamps of one group) at the config-4 / config-5 shapes
mkdir -p gpurun_out
for j in 1 4097; do
HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_c4n8192_j$j.bin HT_TRACE_J1=$j timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check > gpurun_out/tr_c4_$j.log 2>&1
python tools/trace_path.py gpurun_out/tr_c4n8192_j$j.bin >> gpurun_out/trace_paths.txt 2>&1
done
HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_c5n4096_j1.bin HT_TRACE_J1=1 timeout 600 python tools/run_config.py 5 --n 4096 --calls 1 --no-check > gpurun_out/tr_c5.log 2>&1
python tools/trace_path.py gpurun_out/tr_c5n4096_j1.bin >> gpurun_out/trace_paths.txt 2>&1
HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_c2_j1.bin HT_TRACE_J1=1 timeout 600 python tools/run_config.py 2 --calls 1 --no-check > gpurun_out/tr_c2.log 2>&1
python tools/trace_path.py gpurun_out/tr_c2_j1.bin >> gpurun_out/trace_paths.txt 2>&1
