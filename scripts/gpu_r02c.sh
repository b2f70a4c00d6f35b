#!/bin/bash
# round 2: where does k_merge_w's time go on R-MAT 22 -- ncu full capture, column-tile experiment, gather probe
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02c
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
BARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_merge_w -s 2 -c 1 -f \
    -o $O/merge_c2 python bench.py --config 2 $BARGS > $O/ncu_c2.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py $O/merge_c2.ncu-rep --stalls > $O/ncu_merge_c2.txt 2>&1
head -40 $O/ncu_merge_c2.txt
timeout 900 python scripts/exp_coltile.py 2 4 > $O/coltile.txt 2>&1; echo "coltile rc=$?"
cat $O/coltile.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp2 scripts/gather_probe2.cu && timeout 300 /tmp/gp2 22 65241671 > $O/gp2_22.txt 2>&1
cat $O/gp2_22.txt | head -60
