#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
tools/diag/_dispatch_mix > gpurun_out/dispatch_mix.log 2>&1
timeout 900 python -m pytest tests/test_gpu_rng32.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_rng32.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_rng32.log
