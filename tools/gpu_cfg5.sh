#!/bin/bash
# config 5 (the full pipeline) through bench.py, after the mode-1 parity tests
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-cfg5}
timeout 900 python -m pytest tests/test_gpu_rng32.py tests/test_gpu_pipeline.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 ${CFG5_ARGS} > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err
echo "cfg5 rc=$?" >> gpurun_out/bench_cfg5_$TAG.err
