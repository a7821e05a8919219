#!/bin/bash
# Round measurement set: default bench (+ reference arm), its ncu launch list,
# ncu --set full of K1 (config 4 and config 3 nodes, Philox4x32) and of K3
# (config-5 panel set).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-m}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_$TAG.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --no-cpu --no-profile --steps 1 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch_$TAG.log
for c in 4 3; do
  CMD="python bench.py --n-bp 300 --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile --no-parity-mode --config $c"
  $CMD > gpurun_out/plain_k1_${TAG}_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_k1_${TAG}_cfg$c $CMD > gpurun_out/ncu_k1_${TAG}_cfg$c.log 2>&1
  echo "ncu k1 cfg$c rc=$?" >> gpurun_out/ncu_k1_${TAG}_cfg$c.log
done
N_TARGETS=100000 python tools/k3_probe.py > gpurun_out/plain_k3_$TAG.log 2>&1 && \
N_TARGETS=100000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:potential_kernel -s 1 -c 1 -o gpurun_out/prof_k3_$TAG python tools/k3_probe.py > gpurun_out/ncu_k3_$TAG.log 2>&1
echo "ncu k3 rc=$?" >> gpurun_out/ncu_k3_$TAG.log
