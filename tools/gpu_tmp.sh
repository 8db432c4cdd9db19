cd $GRAFT_REPO_ROOT
./tools/rq_bench > gpurun_out/rq_bench.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/k1prof.py 4096 16 16 > gpurun_out/plain_k1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chase -s 100 -c 1 -o gpurun_out/prof_chase_c2_v3 python tools/k1prof.py 4096 16 16 > gpurun_out/ncu_chase.log 2>&1
