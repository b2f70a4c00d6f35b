#!/bin/bash
# merge: A stream (column indices, values, row ends) with an L2 evict-first policy vs without
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03g
mkdir -p $O
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], d['config'].get('algo'), 'step %.4f ms'%d['ms_per_step'], 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  timeout 600 python bench.py --config 2 $BA > $O/c2_ef_$rep.json 2>/dev/null; summ $O/c2_ef_$rep.json c2_ef
  SPMM_LIB=build_variants/libspmm_noef.so timeout 600 python bench.py --config 2 $BA > $O/c2_noef_$rep.json 2>/dev/null; summ $O/c2_noef_$rep.json c2_noef
done
for rep in 1 2; do
  timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_ef_$rep.json 2>/dev/null; summ $O/c4_ef_$rep.json c4_ef
  SPMM_LIB=build_variants/libspmm_noef.so timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_noef_$rep.json 2>/dev/null; summ $O/c4_noef_$rep.json c4_noef
done
timeout 900 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k "regex:k_merge_w" -c 1 --csv python scripts/run_one.py rmat22 64 merge > $O/ncu_ef_c2.csv 2>&1
SPMM_LIB=build_variants/libspmm_noef.so timeout 900 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k "regex:k_merge_w" -c 1 --csv python scripts/run_one.py rmat22 64 merge > $O/ncu_noef_c2.csv 2>&1
grep -h "k_merge_w" $O/ncu_*ef_c2.csv | cut -c1-40,100-400
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat20_n1.csv python scripts/run_one.py rmat20 1 merge folded > /dev/null 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat22_n64.csv python scripts/run_one.py rmat22 64 merge > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "partition or merge or folded or task_queue or bit_identical or accumulate or adversarial or randomized or misaligned or config0" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
timeout 900 python scripts/exp_small_n.py 1,4,16,64 > $O/small_n.txt 2>&1; cat $O/small_n.txt
