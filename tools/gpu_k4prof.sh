#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/analyze_acc.py 3 4000 > gpurun_out/acc_cfg3.log 2>&1
timeout 600 python tools/analyze_acc.py 2 2000 > gpurun_out/acc_cfg2.log 2>&1
CMD="python tools/bench_k4.py 4 4000"
$CMD > gpurun_out/plain_k4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assemble -s 1 -c 1 -o gpurun_out/prof_k4 $CMD > gpurun_out/ncu_k4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k4.log
