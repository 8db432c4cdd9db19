#!/bin/bash
# configs 3 and 4 at their own sizes against the cached oracle samples (oracle_cache/cfg{3,4}.npz,
# written by tools/oracle_cache.py from oracle/ only)
mkdir -p gpurun_out
rm -f gpurun_out/parity_fullsize_c34.jsonl
HT_PARITY_LOG=gpurun_out/parity_fullsize_c34.jsonl timeout 1500 python -m pytest "tests/test_gpu_fullsize.py::test_fullsize_vs_cached_oracle_samples" -q > gpurun_out/parity_c34_test.log 2>&1
echo "rc=$?" >> gpurun_out/parity_c34_test.log
