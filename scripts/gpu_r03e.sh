#!/bin/bash
# folded merge with 16-byte cp.async staging + packed scan flags: parity subset, small-n A/B vs HEAD build
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03e
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "folded or merge_worker or task_queue or bit_identical or accumulate or adversarial or randomized or misaligned or partitions" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
for rep in 1 2; do
  timeout 900 python scripts/exp_small_n.py >> $O/small_n.txt 2>&1
  SPMM_LIB=build_variants/libspmm_head.so timeout 900 python scripts/exp_small_n.py >> $O/small_n.txt 2>&1
done
cat $O/small_n.txt
