#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python tools/shard_scaling.py --config 4 --warmup 2 --steps 2 > gpurun_out/shard_scaling_cfg4.log 2> gpurun_out/shard_scaling_cfg4.err
echo "rc=$?" >> gpurun_out/shard_scaling_cfg4.err
timeout 900 python tools/shard_scaling.py --config 3 --warmup 2 --steps 2 > gpurun_out/shard_scaling_cfg3.log 2> gpurun_out/shard_scaling_cfg3.err
echo "rc=$?" >> gpurun_out/shard_scaling_cfg3.err
