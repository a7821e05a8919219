#!/bin/bash
# A/B of gpurun_variants/ on chosen configs, then ncu --set full of K1 on config 3 / 2 / 4 nodes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
rm -f gpurun_out/ab.log
NOTEST=1 CFGS="${CFGS:-4:20000 3:4000 2:0}" bash tools/gpu_ab.sh
cp gpurun_out/ab.log gpurun_out/ab_${1:-x}.log
for c in ${NCUCFGS:-3 2}; do CFG=$c NBP=300 bash tools/gpu_ncu_wos_cfg.sh k1cfg${c}_${1:-x}; done
