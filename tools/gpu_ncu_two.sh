#!/bin/bash
# ncu --set full of K1 on config-4 and config-3 nodes (one launch each)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-u32}
CFG=4 NBP=300 bash tools/gpu_ncu_wos_cfg.sh k1sph_$TAG
CFG=3 NBP=300 bash tools/gpu_ncu_wos_cfg.sh k1cav_$TAG
