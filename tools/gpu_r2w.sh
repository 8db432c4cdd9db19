#!/bin/bash
mkdir -p gpurun_out
HT_PARITY_LOG=gpurun_out/r2w_parity.jsonl timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2w_pytest.log
timeout 1500 python tools/run_config.py 5 --calls 1 > gpurun_out/r2w_cfg5.json 2> gpurun_out/r2w_cfg5.err
echo "cfg5 rc=$?" >> gpurun_out/r2w_cfg5.err
