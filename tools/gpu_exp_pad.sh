#!/bin/bash
# Session-5 A/B: chain shared-memory strides (default: conflict-free pads; tools/libht_pad8.so: the old +8)
mkdir -p gpurun_out
L=gpurun_out/exp_pad.log
: > $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/exp_pad_suite.log 2>&1
echo "suite rc=$?" >> gpurun_out/exp_pad_suite.log
for c in 4 3 2; do
  echo "== config $c new pads" >> $L
  timeout 900 python tools/run_config.py $c --calls 2 >> $L 2>&1
  echo "== config $c pad 8 (old)" >> $L
  timeout 900 python tools/run_config.py $c --lib tools/libht_pad8.so --calls 2 --no-check >> $L 2>&1
done
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for v in new pad8; do
  lib=""; [ $v = pad8 ] && lib="--lib tools/libht_pad8.so"
  timeout 900 ncu --metrics $M --clock-control none -k regex:chain_kernel -s 40 -c 8 --csv --log-file gpurun_out/exp_pad_ncu_$v.csv python tools/run_config.py 4 --n 4096 --calls 0 --no-check $lib > gpurun_out/exp_pad_ncu_$v.log 2>&1
done
echo "== config 5 new pads" >> $L
timeout 1500 python tools/run_config.py 5 --calls 1 >> $L 2>&1
echo "== config 4 new pads HT_WY=1" >> $L
HT_WY=1 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
echo "== config 4 new pads HT_QZ_STREAM=1" >> $L
HT_QZ_STREAM=1 timeout 900 python tools/run_config.py 4 --calls 2 >> $L 2>&1
echo "== config 3 new pads HT_QZ_STREAM=1" >> $L
HT_QZ_STREAM=1 timeout 900 python tools/run_config.py 3 --calls 2 >> $L 2>&1
