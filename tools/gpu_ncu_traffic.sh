#!/bin/bash
# DRAM bytes of one full config-4 K1 launch (the roofline 'traffic' field)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:wos_nodes -c 1 --csv $CMD > gpurun_out/ncu_traffic_${1:-r1}.csv 2> gpurun_out/ncu_traffic_${1:-r1}.err
echo "rc=$?" >> gpurun_out/ncu_traffic_${1:-r1}.err
