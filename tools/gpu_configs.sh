#!/bin/bash
# configs 1, 2, 3 (full) and 5 (full) through bench.py
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-cfgs}
for c in 1 2 3; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_cfg${c}_$TAG.json 2> gpurun_out/bench_cfg${c}_$TAG.err
  echo "cfg$c rc=$?" >> gpurun_out/bench_cfg${c}_$TAG.err
done
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 ${CFG5_ARGS} > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err
echo "cfg5 rc=$?" >> gpurun_out/bench_cfg5_$TAG.err
