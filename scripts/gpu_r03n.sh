#!/bin/bash
# lane-folded merge with float2 slots (n = 2, 6, 10..): folded parity subset, small-n A/B vs the previous build
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03n
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "folded or merge_worker or task_queue or bit_identical or accumulate or config0 or adversarial" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
for rep in 1 2; do
  timeout 900 python scripts/exp_small_n.py 2,6,10,4,1 >> $O/small_n.txt 2>&1
  SPMM_LIB=build_variants/libspmm_nof2.so timeout 900 python scripts/exp_small_n.py 2,6,10,4,1 >> $O/small_n.txt 2>&1
done
cat $O/small_n.txt
