#!/bin/bash
# K1 A/B on one box: pytest subset (TESTS), then bench.py per (rng, library)
# variant (VARIANTS="rng:lib ...", lib relative to the repo) and config
# (CFGS="config:n_bp ..."), then (NCU=1) ncu --set full of K1 per rng.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-rng}
L=paper_1210_1491_b200/_lib/libbiewos_b200.so
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
for cn in ${CFGS:-4:20000 3:4000 2:0}; do
  cfg=${cn%%:*}; nbp=${cn##*:}
  for v in ${VARIANTS:-64:$L 32:$L}; do
    r=${v%%:*}; lib=${v#*:}
    BW_LIB_PATH=$PWD/$lib timeout 300 python bench.py --n-bp $nbp --steps 2 --warmup 1 --no-cpu --no-e2e --config $cfg --rng $r 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('cfg$cfg rng$r', '$lib'.split('/')[-1], '%.4g' % d['value'], '%.1f ms' % d['ms_per_step'], d['clocks']['sm_mhz'], d['neumann_check'])
    elif 'Error' in l or 'error' in l: print(l.strip())" >> gpurun_out/ab_$TAG.log
  done
done
if [ -n "$NCU" ]; then
for r in ${NCU_RNGS:-64 32}; do
  CMD="python bench.py --n-bp 300 --steps 1 --warmup 1 --no-cpu --no-e2e --rng $r --config ${NCU_CFG:-4}"
  $CMD > gpurun_out/plain_ncu_${TAG}_$r.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wos_nodes -c 1 -o gpurun_out/prof_k1_${TAG}_$r $CMD > gpurun_out/ncu_k1_${TAG}_$r.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_k1_${TAG}_$r.log
done
fi
