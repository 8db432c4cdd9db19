#!/bin/bash
# config 3 at its own size: the oracle on the box's host cores (tools/oracle_cache.py, oracle/ only),
# then the GPU parity test against its cached samples
mkdir -p gpurun_out
timeout 5000 python tools/oracle_cache.py 3 > gpurun_out/oracle_cfg3.log 2>&1
cp oracle_cache/cfg3.npz gpurun_out/ 2>/dev/null
HT_PARITY_LOG=gpurun_out/parity_fullsize_c3.jsonl timeout 900 python -m pytest "tests/test_gpu_fullsize.py::test_fullsize_vs_cached_oracle_samples[3]" -x -q > gpurun_out/parity_c3_test.log 2>&1
echo "rc=$?" >> gpurun_out/parity_c3_test.log
