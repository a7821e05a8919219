#!/bin/bash
# Philox4x32 two-steps-per-block stream: stream/walk parity tests, then the A/B
# of the variants in gpurun_variants/ on configs 4, 3 and 2.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rng32.py tests/test_gpu_wos.py tests/test_gpu_strata.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_u32.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_u32.log
rm -f gpurun_out/ab.log
NOTEST=1 CFGS="${CFGS:-4:20000 3:4000 2:0}" bash tools/gpu_ab.sh
cp gpurun_out/ab.log gpurun_out/ab_u32.log
