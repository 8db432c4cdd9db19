#!/bin/bash
# helper-count A/B at config 4 (full size) and the n=8192 critical path with 3 helpers per sweep
mkdir -p gpurun_out
for h in 2 3 1; do
HT_HELPERS=$h timeout 600 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/hel_c4_h$h.json 2>&1
done
HT_HELPERS=3 HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_c4n8192_h3.bin timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check > /dev/null 2>&1
python tools/trace_path.py gpurun_out/tr_c4n8192_h3.bin > gpurun_out/trace_h3.txt 2>&1
