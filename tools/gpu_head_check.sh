#!/bin/bash
# HEAD validation: GPU tests, smoke, default bench + cfg3 line.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-head}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/bench_cfg3_$TAG.json 2> gpurun_out/bench_cfg3_$TAG.err
echo "cfg3 rc=$?" >> gpurun_out/bench_cfg3_$TAG.err
