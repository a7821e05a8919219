#!/bin/bash
# A/B of library variants on one box: tests on the default build, then bench per variant
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu_ab.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab.log
for lib in paper_1210_1491_b200/_lib/libbiewos_b200.so gpurun_variants/*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  BW_LIB_PATH=$PWD/$lib timeout 300 python bench.py --n-bp ${NBP:-10000} --steps 2 --warmup 1 --no-cpu --no-e2e --config ${CFG:-4} 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])
    else: print(l.strip())" >> gpurun_out/ab.log
done
