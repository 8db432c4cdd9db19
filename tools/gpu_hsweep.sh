#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/k1prof.log
for a in "8192 64 32" "4096 16 32"; do
  for hh in 1 2 3; do
    echo "== $a H=$hh" >> gpurun_out/k1prof.log
    HT_HELPERS=$hh timeout 600 python tools/k1prof.py $a 2>&1 | grep wall | tail -1 >> gpurun_out/k1prof.log
  done
done
