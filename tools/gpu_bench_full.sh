#!/bin/bash
# Full default bench (the driver's command) + its ncu launch list.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-full}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_$TAG.err
if [ -n "$LAUNCHES" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_launch_$TAG.log
fi
