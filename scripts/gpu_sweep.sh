#!/bin/bash
# tuning sweep: bench each library variant on CASES (see scripts/sweep.py); optional ncu capture
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout ${SWEEP_TIMEOUT:-1500} python scripts/sweep.py paper_1803_08601_b200/libspmm.so $(ls build_variants/*.so 2>/dev/null) > gpurun_out/sweep_${TAG:-x}.txt 2>&1
if [ -n "$NCU_CFG" ]; then CFG=$NCU_CFG ALGO=${NCU_ALGO:-auto} TAG=${TAG:-x} bash scripts/gpu_prof1.sh; python scripts/ncu_summary.py gpurun_out/prof_${TAG:-x}.ncu-rep --stalls > gpurun_out/ncu_${TAG:-x}.txt 2>&1; fi
cat gpurun_out/sweep_${TAG:-x}.txt
