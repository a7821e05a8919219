#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for lib in paper_1210_1491_b200/_lib/libbiewos_b200.so gpurun_variants/*.so; do
  echo "== $lib" >> gpurun_out/k4.log
  BW_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_k4.py 4 20000 >> gpurun_out/k4.log 2>&1
  BW_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_k4.py 3 20000 >> gpurun_out/k4.log 2>&1
done
echo "== cfg3 pruned grid" >> gpurun_out/k4.log
timeout 600 python bench.py --config 3 --n-bp 4000 --steps 1 --warmup 1 --no-cpu --no-e2e >> gpurun_out/k4.log 2>&1
