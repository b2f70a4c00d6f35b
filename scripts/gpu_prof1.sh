#!/bin/bash
# one ncu --set full capture of k_tile for a given bench config: CFG, ALGO, TAG, LIB
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export SPMM_LIB=${LIB:-$PWD/paper_1803_08601_b200/libspmm.so}
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 1 -f \
  -o gpurun_out/prof_${TAG} python bench.py --config ${CFG:-1} --algo ${ALGO:-auto} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1
tail -n 2 gpurun_out/ncu_${TAG}.log
