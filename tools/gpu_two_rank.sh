#!/bin/bash
# The N > 1 path of bench.py on a one-GPU box: two ranks share the device over
# gloo (BW_BENCH_BACKEND); walk-step totals must equal the one-rank run.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
A="--n-bp ${NBP:-4000} --steps 2 --warmup 1 --no-cpu --config ${CFG:-4}"
timeout 600 python bench.py $A > gpurun_out/two_rank_n1.json 2> gpurun_out/two_rank_n1.err
echo "n1 rc=$?" >> gpurun_out/two_rank_n1.err
BW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 $A > gpurun_out/two_rank_n2.json 2> gpurun_out/two_rank_n2.err
echo "n2 rc=$?" >> gpurun_out/two_rank_n2.err
