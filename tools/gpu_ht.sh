#!/bin/bash
# H/T apply-chain timing (no Q/Z) for a few shapes -- dev helper
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/ht.log
for a in $HTARGS; do
  echo "== $a" >> gpurun_out/ht.log
  timeout 300 python tools/k1prof.py ${a//,/ } 2>&1 | grep wall | tail -1 >> gpurun_out/ht.log
done
echo done
