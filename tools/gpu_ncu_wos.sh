#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --n-bp 300 --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain_ncu.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_wos_${1:-r1a} $CMD > gpurun_out/ncu_wos.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_wos.log
