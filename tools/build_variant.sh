#!/bin/bash
# Build the library with extra -D flags into gpurun_variants/NAME.so (for tools/gpu_ab.sh)
# usage: tools/build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p gpurun_variants
C=paper_1210_1491_b200/csrc
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared "$@" \
  -o gpurun_variants/$name.so $C/bw_capi.cu $C/bw_wos.cu $C/bw_potential.cu $C/bw_lu.cu $C/bw_diag.cu \
  $C/bw_patch.cu $C/bw_point.cu $C/bw_lp.cu $C/bw_dtn_class.cu $C/bw_patch_large.cu $C/bw_group.cu -ldl
