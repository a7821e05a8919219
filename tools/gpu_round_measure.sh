#!/bin/bash
# One box, the whole measurement set of a round: GPU tests + smoke, the driver's
# default bench + reference arm + ncu launch list, configs 1/2/3/5, and ncu --set
# full of K1 (config-4 nodes) and of K1 on the cavity scene (config 3).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-r1}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
LAUNCHES=1 bash tools/gpu_bench_full.sh $TAG
bash tools/gpu_configs.sh $TAG
bash tools/gpu_ncu_wos.sh $TAG
CMD3="python bench.py --config 3 --n-bp 200 --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD3 > gpurun_out/plain_ncu3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_wos3_$TAG $CMD3 > gpurun_out/ncu_wos3.log 2>&1
echo "ncu3 rc=$?" >> gpurun_out/ncu_wos3.log
