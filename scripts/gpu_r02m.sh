#!/bin/bash
# round 2: tiled kernel with TMA B blocks -- parity + density sweep
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02m
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiled" > $O/pytest_tiled.log 2>&1; echo "rc=$?" >> $O/pytest_tiled.log
tail -3 $O/pytest_tiled.log
timeout 2400 python scripts/density_sweep.py --pcts 0.1,1,5,12,20 --out $O/density_sweep > $O/density.log 2>&1; echo "density rc=$?"
cat $O/density.log | tail -8
