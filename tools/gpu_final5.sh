#!/bin/bash
# Session-5 final: new defaults (conflict-free chain strides, Q/Z evict-first, WY from r = 64)
mkdir -p gpurun_out
L=gpurun_out/final5.log
: > $L
echo "== config 4 defaults" >> $L
timeout 900 python tools/run_config.py 4 --calls 2 >> $L 2>&1
echo "== config 4 HT_WY=0" >> $L
HT_WY=0 timeout 900 python tools/run_config.py 4 --calls 2 --no-check >> $L 2>&1
bash tools/gpu_check.sh
cp gpurun_out/bench_c4.json gpurun_out/final5_bench_c4.json
timeout 900 python bench.py --config 3 > gpurun_out/final5_bench_c3.json 2> gpurun_out/final5_bench_c3.err
timeout 600 python bench.py --config 2 > gpurun_out/final5_bench_c2.json 2> gpurun_out/final5_bench_c2.err
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for v in new pad8; do
  lib=""; [ $v = pad8 ] && lib="--lib tools/libht_pad8.so"
  HT_WY=0 timeout 900 ncu --metrics $M --clock-control none -k regex:chain_kernel -s 40 -c 8 --csv --log-file gpurun_out/final5_ncu_bank_$v.csv python tools/run_config.py 4 --n 4096 --calls 1 --no-check $lib > gpurun_out/final5_ncu_$v.log 2>&1
done
