#!/bin/bash
# round 2: L2 priority by popularity on the R-MAT gather pattern (probe), scales 22 and 26
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02e
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp3 scripts/gather_probe3.cu
timeout 600 /tmp/gp3 26 268435456 policy > $O/gp3_pol26.txt 2>&1
timeout 300 /tmp/gp3 22 65241671 policy > $O/gp3_pol22.txt 2>&1
cat $O/gp3_pol26.txt $O/gp3_pol22.txt
