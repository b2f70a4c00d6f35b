#!/bin/bash
# folded merge at n = 1 on R-MAT 20 (launch list + full capture); row split 8 x 4 groups for n > 96:
# parity subset and banded n = 128 bench
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03d
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config0 or tiled or padding or b_staging or randomized or misaligned or every_row or bit_identical" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
timeout 600 python bench.py --config 1 --n 128 --no-extras --no-e2e --no-cpu-baseline > $O/c1_n128.json 2>/dev/null
python -c "import json;d=json.load(open('$O/c1_n128.json'));r=d['roofline'];print('c1 n128', r['avg_launch_ms'], r['frac'])"
timeout 300 python scripts/run_one.py rmat20 1 merge folded > $O/run_one.txt 2>&1; echo "run_one rc=$?"; tail -2 $O/run_one.txt
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat20_n1.csv python scripts/run_one.py rmat20 1 merge folded > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k "regex:k_merge_f" -s 1 -c 1 -f -o $O/prof_merge_f_rmat20_n1 python scripts/run_one.py rmat20 1 merge folded > /dev/null 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py $O/prof_merge_f_rmat20_n1.ncu-rep --stalls > $O/ncu_merge_f_rmat20_n1.txt 2>&1; head -40 $O/ncu_merge_f_rmat20_n1.txt
