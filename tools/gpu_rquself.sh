#!/bin/bash
# HT_RQU_SELF A/B at config 4 (full size), traces at n=8192, parity with the share on
mkdir -p gpurun_out
HT_RQU_SELF=1/2 timeout 900 python -m pytest tests/test_gpu_rqu.py tests/test_gpu_parity.py -x -q > gpurun_out/self_parity.log 2>&1
echo "rc=$?" >> gpurun_out/self_parity.log
for s in 0/1 1/3 1/2 2/3; do
tag=$(echo $s | tr / _)
HT_RQU_SELF=$s timeout 600 python tools/run_config.py 4 --calls 2 --no-check > gpurun_out/self_c4_$tag.json 2>&1
HT_RQU_SELF=$s HT_LAG_CHECK=1 HT_TRACE_DUMP=gpurun_out/tr_self_$tag.bin timeout 600 python tools/run_config.py 4 --n 8192 --calls 1 --no-check > /dev/null 2>&1
echo "== $s" >> gpurun_out/trace_self.txt
python tools/trace_path.py gpurun_out/tr_self_$tag.bin >> gpurun_out/trace_self.txt 2>&1
done
