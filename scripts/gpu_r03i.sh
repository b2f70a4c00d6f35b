#!/bin/bash
# n = 128 row groups by mean row length (8 x 4 up to d = 64) + refit guard: quick check
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "refit or config0 or b_staging or padding or randomized or tiled" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
timeout 1200 python scripts/sweep_config4.py --ns 128 --out $O/config3_n128 > $O/config3_n128.log 2>&1; echo "sweep rc=$?"; tail -3 $O/config3_n128.log
