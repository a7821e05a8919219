#!/bin/bash
# GPU tests on the bounds-checked build (-DBW_CHECKS=1), the stand-in for compute-sanitizer
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
BW_LIB_PATH=$PWD/gpurun_variants/checked.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs --deselect tests/test_gpu_integration.py > gpurun_out/pytest_gpu_checked.log 2>&1
echo "pytest checked rc=$?" >> gpurun_out/pytest_gpu_checked.log
BW_LIB_PATH=$PWD/gpurun_variants/checked.so timeout 600 python bench.py --config 3 --n-bp 2000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/bench_cfg3_checked.json 2> gpurun_out/bench_cfg3_checked.err
echo "cfg3 checked rc=$?" >> gpurun_out/bench_cfg3_checked.err
