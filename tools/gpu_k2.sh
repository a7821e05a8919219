#!/bin/bash
# K2 A/B: tests, timings of the product library and of gpurun_variants/lu_old.so,
# bitwise comparison of their outputs, ncu of the new kernel.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_potential_lu.py tests/test_gpu_dtn.py tests/test_gpu_cpp.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_k2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k2.log
rm -f gpurun_out/k2_ab.log
for cfgs in "54 100000 2" "54 20000 7" "64 20000 8" "33 20000 1" "5 20000 2" "1 1000 1"; do
  set -- $cfgs
  for lib in paper_1210_1491_b200/_lib/libbiewos_b200.so gpurun_variants/lu_old.so; do
    [ -f $lib ] || continue
    tag=$(basename $lib .so)
    echo -n "$tag " >> gpurun_out/k2_ab.log
    BW_LIB_PATH=$PWD/$lib timeout 300 python tools/bench_k2.py $1 $2 $3 /tmp/k2_${tag}_$1_$3.npz >> gpurun_out/k2_ab.log 2>&1
  done
  python - >> gpurun_out/k2_ab.log 2>&1 <<PY
import numpy as np, os
a='/tmp/k2_libbiewos_b200_$1_$3.npz'; b='/tmp/k2_lu_old_$1_$3.npz'
if os.path.exists(a) and os.path.exists(b):
    A, B = np.load(a), np.load(b)
    print('bitwise m=$1 nrhs=$3:', {k: bool(np.array_equal(A[k].view(np.uint8), B[k].view(np.uint8))) for k in ('X', 'resid', 'info')})
PY
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lu_kernel -c 1 -o gpurun_out/prof_k2 python tools/bench_k2.py 54 100000 2 > gpurun_out/ncu_k2.log 2>&1
fi
