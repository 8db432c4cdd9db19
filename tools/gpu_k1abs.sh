#!/bin/bash
# per-step K1 phase cycles for chosen sweeps (HT_K1PROF_T) -- dev helper
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/k1abs.log
for a in $K1ARGS; do
  for tt in $K1T; do
    echo "== $a t0=$tt" >> gpurun_out/k1abs.log
    HT_K1PROF=1 HT_K1PROF_T=$tt timeout 300 python tools/k1prof.py ${a//,/ } 2>&1 | grep -E "K1 cycles|wall" >> gpurun_out/k1abs.log
  done
done
echo done
