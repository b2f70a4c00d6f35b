#!/bin/bash
# round 2: tiled kernel (NEXT-4) parity + density sweep; folded timing with the queued-task floor
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02l
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiled or heuristic or auto" > $O/pytest_tiled.log 2>&1; echo "rc=$?" >> $O/pytest_tiled.log
tail -15 $O/pytest_tiled.log
timeout 2400 python scripts/density_sweep.py --pcts 0.1,0.5,1,2,5,9,12,15,20 --out $O/density_sweep > $O/density.log 2>&1; echo "density rc=$?"
cat $O/density.log | tail -14
timeout 900 python scripts/exp_fold.py 1,4,16 > $O/exp_fold.txt 2>&1
cat $O/exp_fold.txt
