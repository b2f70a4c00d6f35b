#!/bin/bash
# k_partition as one coalesced pass over the rows + k_fixup with its loads issued up front: parity
# (partition vs oracle, merge families), config 2 / 4 step times and small-n AUTO vs the previous build
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03f
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -m gpu -q -x -k "partition or merge or folded or task_queue or bit_identical or accumulate or adversarial or randomized or misaligned or config0 or every_row or rmat or dist or row_blocks or fused or iterative" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], d['config'].get('algo'), 'step %.4f ms'%d['ms_per_step'], 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  timeout 600 python bench.py --config 2 $BA > $O/c2_new_$rep.json 2>/dev/null; summ $O/c2_new_$rep.json c2_new
  SPMM_LIB=build_variants/libspmm_head.so timeout 600 python bench.py --config 2 $BA > $O/c2_head_$rep.json 2>/dev/null; summ $O/c2_head_$rep.json c2_head
done
timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_new.json 2>/dev/null; summ $O/c4_new.json c4_new
timeout 900 python scripts/exp_small_n.py 1,4,16,64 >> $O/small_n.txt 2>&1
SPMM_LIB=build_variants/libspmm_head.so timeout 900 python scripts/exp_small_n.py 1,4,16,64 >> $O/small_n.txt 2>&1
cat $O/small_n.txt
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat20_n1.csv python scripts/run_one.py rmat20 1 merge folded > /dev/null 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat22_n64.csv python scripts/run_one.py rmat22 64 merge > /dev/null 2>&1
grep -h "k_partition\|k_fixup" $O/launches_*.csv | cut -c1-200 | tail -8
