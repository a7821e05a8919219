#!/bin/bash
# ncu --set full of the K7 kernels (class_apply, class_h, class_geom) on a config-4 run
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-k7}
CMD="python bench.py --n-bp ${NBP:-4000} --steps 1 --warmup 1 --no-cpu --no-e2e --config ${CFG:-4}"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:class_ -c 3 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
