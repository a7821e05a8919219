#!/bin/bash
# A/B of library variants in the parity mode (--rng 64)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
rm -f gpurun_out/ab64.log
for cn in ${CFGS:-4:10000 3:2000 2:0}; do
  cfg=${cn%%:*}; nbp=${cn##*:}
  for lib in paper_1210_1491_b200/_lib/libbiewos_b200.so gpurun_variants/*.so; do
    BW_LIB_PATH=$PWD/$lib timeout 300 python bench.py --rng 64 --n-bp $nbp --steps 2 --warmup 1 --no-cpu --no-e2e --no-profile --config $cfg 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('cfg$cfg', '$lib'.split('/')[-1], '%.4g' % d['value'], '%.1f ms' % d['ms_per_step'], d['clocks']['sm_mhz'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/ab64.log
  done
done
