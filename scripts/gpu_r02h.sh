#!/bin/bash
# round 2: folded merge v2 (slot starts from a row-end scan) -- parity + timing
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02h
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "worker or folded or queue or config0 or adversarial or partitions or identical" > $O/pytest_fold.log 2>&1; echo "rc=$?" >> $O/pytest_fold.log
tail -4 $O/pytest_fold.log
timeout 1200 python scripts/exp_fold.py 1,4,16 > $O/exp_fold.txt 2>&1; echo "exp rc=$?"
cat $O/exp_fold.txt
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_merge_f -s 1 -c 1 -f \
    -o $O/mf_rmat20 python scripts/run_one.py rmat20 1 merge folded 1 > $O/ncu_rmat20.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py $O/mf_rmat20.ncu-rep --stalls > $O/ncu_mf_rmat20.txt 2>&1
head -50 $O/ncu_mf_rmat20.txt
