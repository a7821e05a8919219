#!/bin/bash
# Round-2 validation: GPU tests on the product library and on the bounds-checked
# build (the stand-in for compute-sanitizer), smoke, default bench + reference
# arm, configs 1/2/3 and 5.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-r2}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
BW_LIB_PATH=$PWD/gpurun_variants/checked.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs --deselect tests/test_gpu_integration.py > gpurun_out/pytest_gpu_checked_$TAG.log 2>&1
echo "pytest checked rc=$?" >> gpurun_out/pytest_gpu_checked_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_$TAG.err
for c in 1 2 3; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/bench_cfg${c}_$TAG.json 2> gpurun_out/bench_cfg${c}_$TAG.err
  echo "cfg$c rc=$?" >> gpurun_out/bench_cfg${c}_$TAG.err
done
timeout 1500 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err
echo "cfg5 rc=$?" >> gpurun_out/bench_cfg5_$TAG.err
