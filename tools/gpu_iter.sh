#!/bin/bash
# Iteration loop on the box: GPU tests + small bench (+ optional ncu of the WOS kernel)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
CMD="python bench.py --n-bp ${NBP:-10000} --steps 2 --warmup 1 --no-cpu --no-e2e --config ${CFG:-4}"
$CMD > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
if [ -n "$NCU" ]; then
  CMD2="python bench.py --n-bp 300 --steps 1 --warmup 1 --no-cpu --no-e2e --config ${CFG:-4}"
  $CMD2 > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_$TAG $CMD2 > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
fi
