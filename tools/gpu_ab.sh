#!/bin/bash
# A/B of library variants on one box: GPU tests on the default build, then a short
# bench per variant and config. CFGS="4:20000 3:4000 2:0" (config:n_bp, 0 = full)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu_ab.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab.log
fi
for cn in ${CFGS:-4:20000 3:4000 2:0}; do
  cfg=${cn%%:*}; nbp=${cn##*:}
  for lib in paper_1210_1491_b200/_lib/libbiewos_b200.so gpurun_variants/*.so; do
    BW_LIB_PATH=$PWD/$lib timeout 300 python bench.py --n-bp $nbp --steps 2 --warmup 1 --no-cpu --no-e2e --config $cfg 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('cfg$cfg', '$lib'.split('/')[-1], '%.4g' % d['value'], '%.1f ms' % d['ms_per_step'], d['clocks']['sm_mhz'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/ab.log
  done
done
