#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over a subset of the GPU parity tests and smoke()
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="config0_parity and (f32_plus_times or i32_min_plus) and (64 or 1-) or b_staging_parity and aligned-64 or misaligned_csr_views and banded or row_pairing_parity and banded_odd or merge_partitions"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -n 4 gpurun_out/sanitize_$tool.log
done
