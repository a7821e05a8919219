#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_sweep.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sweep.log
run() { timeout 600 python bench.py "$@" --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(round(d['value']/1e9,2),'Gsteps/s', round(d['ms_per_step']), 'ms k1', round(d['k1_share_of_step'],4), d['neumann_check'])
    else: print(l.strip()[:200])"; }
echo "== cfg4 10k" >> gpurun_out/sweep.log; run --n-bp 10000 >> gpurun_out/sweep.log
for g in ${GRIDS:-8 12 16 20 24 32}; do echo "== cfg3 4k grid $g" >> gpurun_out/sweep.log; BW_CAVITY_GRID=$g run --config 3 --n-bp 4000 >> gpurun_out/sweep.log; done
