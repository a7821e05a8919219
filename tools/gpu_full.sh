#!/bin/bash
# The round's validation set on one box: every GPU test, smoke(), the driver's
# default bench (B200 arm and reference arm), and config 5 (CFG5=1).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-full}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_$TAG.err
if [ -n "$CFG5" ]; then
  timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err
  echo "cfg5 rc=$?" >> gpurun_out/bench_cfg5_$TAG.err
fi
