#!/bin/bash
# round 2: ncu of the lane-folded merge kernel (R-MAT 20, lognormal, n = 1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02g
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for m in rmat20 lognormal; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_merge_f -s 1 -c 1 -f \
    -o $O/mf_$m python scripts/run_one.py $m 1 merge folded 1 > $O/ncu_$m.log 2>&1; echo "ncu $m rc=$?"
  python scripts/ncu_summary.py $O/mf_$m.ncu-rep --stalls > $O/ncu_mf_$m.txt 2>&1
  head -60 $O/ncu_mf_$m.txt
done
