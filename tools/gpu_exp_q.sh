#!/bin/bash
# Session-5 A/B: helpers per sweep vs group width at config 4 (and the chase alone, no Q/Z)
mkdir -p gpurun_out
L=gpurun_out/exp_q.log
: > $L
echo "== noqz helpers=2 (default)" >> $L
timeout 600 python tools/noqz_prof.py 4 16384 0 >> $L 2>&1
echo "== noqz helpers=3" >> $L
HT_HELPERS=3 timeout 600 python tools/noqz_prof.py 4 16384 0 >> $L 2>&1
for q in 24 28; do
  echo "== config 4 q=$q" >> $L
  timeout 900 python tools/run_config.py 4 --q $q --calls 2 >> $L 2>&1
done
echo "== config 4 q=32 (default)" >> $L
timeout 900 python tools/run_config.py 4 --calls 2 >> $L 2>&1
echo "== config 5 q=24" >> $L
timeout 1500 python tools/run_config.py 5 --q 24 --calls 1 --no-check >> $L 2>&1
