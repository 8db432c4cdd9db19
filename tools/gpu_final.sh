#!/bin/bash
# round-end evidence: full GPU test suite, bench lines of configs 1-4 and the reference arm,
# the launch list of the default bench command and one ncu --set full capture of the top kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_fullbench.sh
bash tools/gpu_profile_final.sh
echo done
