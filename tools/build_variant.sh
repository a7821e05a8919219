#!/bin/bash
# Build the library with extra -D flags into gpurun_variants/NAME.so (for tools/gpu_ab.sh)
# usage: tools/build_variant.sh NAME -DFOO=1 ...
# Sources compile in parallel into a scratch object directory.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p gpurun_variants
C=paper_1210_1491_b200/csrc
O=$(mktemp -d /tmp/bwvar.XXXXXX)
pids=()
for s in bw_capi bw_wos bw_potential bw_lu bw_diag bw_patch bw_point bw_lp bw_dtn_class bw_patch_large bw_group; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" \
    -c $C/$s.cu -o $O/$s.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpurun_variants/$name.so $O/*.o -ldl
rm -rf $O
echo gpurun_variants/$name.so
