#!/bin/bash
# round 2: tiled kernel variants (U = 4; 1 CTA/SM at 255 registers; U = 4 + TMA) on the density sweep
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02o
mkdir -p $O
for v in tl_u4 tl_b1 tl_u4tma; do
  SPMM_LIB=$PWD/build_variants/lib_$v.so timeout 1200 python scripts/density_sweep.py --pcts 0.1,1,5,12 --out $O/density_$v > $O/density_$v.log 2>&1
  echo "== $v"; tail -6 $O/density_$v.log
done
