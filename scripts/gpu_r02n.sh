#!/bin/bash
# round 2: tiled kernel with cached row batches -- parity + density sweep (cp.async and TMA B blocks)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02n
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiled" > $O/pytest_tiled.log 2>&1; echo "rc=$?" >> $O/pytest_tiled.log
tail -3 $O/pytest_tiled.log
timeout 2400 python scripts/density_sweep.py --pcts 0.1,1,5,12,20 --out $O/density_sweep > $O/density.log 2>&1; echo "density rc=$?"
cat $O/density.log | tail -7
SPMM_LIB=$PWD/build_variants/lib_tltma.so timeout 2400 python scripts/density_sweep.py --pcts 0.1,1,5,12,20 --out $O/density_sweep_tma > $O/density_tma.log 2>&1; echo "density tma rc=$?"
cat $O/density_tma.log | tail -7
