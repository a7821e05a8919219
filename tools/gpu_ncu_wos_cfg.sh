#!/bin/bash
# ncu --set full of K1 on a chosen config (default: cfg3 cavities)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-k1cav}
CMD="python bench.py --n-bp ${NBP:-300} --steps 1 --warmup 1 --no-cpu --no-e2e --config ${CFG:-3}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
