#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
BW_WOS_SLOTS=2 timeout 600 python -m pytest tests/test_gpu_wos.py tests/test_gpu_dtn.py -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_slots2.log 2>&1
echo "pytest slots2 rc=$?" >> gpurun_out/pytest_slots2.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu_ab2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab2.log
for cfg in "1 paper_1210_1491_b200/_lib/libbiewos_b200.so" "2 paper_1210_1491_b200/_lib/libbiewos_b200.so" "2 gpurun_variants/lib_s2b5.so"; do
  set -- $cfg
  echo "== slots=$1 $2" >> gpurun_out/ab2.log
  BW_WOS_SLOTS=$1 BW_LIB_PATH=$PWD/$2 timeout 300 python bench.py --n-bp 10000 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['k1_share_of_step'], d['neumann_check'])
    else: print(l.strip()[:200])" >> gpurun_out/ab2.log
done
