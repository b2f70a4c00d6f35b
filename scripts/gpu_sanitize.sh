#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over a subset of the GPU parity tests: config 0 in
# two kinds, B staging, misaligned CSR views, both merge partitions, both merge workers (whole warp,
# lane-folded) with the task queue, R-MAT merge cases, the execute epilogue and the column split.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=${O:-gpurun_out/sanitize}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="config0_parity and (f32_plus_times or i32_min_plus) and (64 or 1-) or b_staging_parity and aligned-64 or misaligned_csr_views and banded or merge_partitions or (merge_worker_parity and rmat12 and (f32_plus_times or i32_min_plus) and (1- or 16-)) or merge_task_queue or (execute_accumulate and i32_min_plus and 16) or split_columns_kernel and rmat12"
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.log
  tail -n 4 $O/sanitize_$tool.log
done
