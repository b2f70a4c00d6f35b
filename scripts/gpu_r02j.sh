#!/bin/bash
# round 2: folded-merge tuning variants + compute-sanitizer over the new kernels
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02j
mkdir -p $O
for v in l16t64 l4b12; do
  SPMM_LIB=$PWD/build_variants/lib_$v.so timeout 900 python scripts/exp_fold.py 1,4,16 > $O/exp_fold_$v.txt 2>&1
  echo "== $v"; cat $O/exp_fold_$v.txt
done
O=gpurun_out/r02j bash scripts/gpu_sanitize.sh
