#!/bin/bash
# quick GPU iteration: parity tests, k1 profile, short bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/k1prof.log
for a in $K1ARGS; do
  echo "== $a" >> gpurun_out/k1prof.log
  HT_K1PROF=1 timeout 300 python tools/k1prof.py ${a//,/ } >> gpurun_out/k1prof.log 2>&1
done
for c in $BENCHCFG; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
echo done
