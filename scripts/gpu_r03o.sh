#!/bin/bash
# lane-folded merge, 1-2 lanes per slot: L = 4 (default) vs 5 / 6 items per slot per chunk
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03o
mkdir -p $O
for v in l5 l6; do
  SPMM_LIB=build_variants/libspmm_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "folded or (merge_worker and folded)" > $O/pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 $O/pytest_$v.log
done
for rep in 1 2; do
  timeout 900 python scripts/exp_small_n.py 1,2,4,8 >> $O/small_n.txt 2>&1
  for v in l5 l6; do SPMM_LIB=build_variants/libspmm_$v.so timeout 900 python scripts/exp_small_n.py 1,2,4,8 >> $O/small_n.txt 2>&1; done
done
cat $O/small_n.txt
