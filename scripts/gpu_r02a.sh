#!/bin/bash
# round 2, first look at k_merge_w: merge parity subset, bench configs 2/4 over build variants, full GPU suite
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out/r02a
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "merge or adversarial or config0 or empty or partition" > $O/pytest_merge.log 2>&1; echo "rc=$?" >> $O/pytest_merge.log
tail -3 $O/pytest_merge.log
BA="--steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for v in default mb5 mb4u16 tile; do
  if [ $v = default ]; then export SPMM_LIB=$PWD/paper_1803_08601_b200/libspmm.so; else export SPMM_LIB=$PWD/build_variants/lib_$v.so; fi
  timeout 300 python bench.py --config 2 $BA > $O/b2_$v.json 2> $O/b2_$v.err
  echo "$v c2: $(python -c "import json;d=json.load(open('$O/b2_$v.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
for v in default mb5 tile; do
  if [ $v = default ]; then export SPMM_LIB=$PWD/paper_1803_08601_b200/libspmm.so; else export SPMM_LIB=$PWD/build_variants/lib_$v.so; fi
  timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b4_$v.json 2> $O/b4_$v.err
  echo "$v c4: $(python -c "import json;d=json.load(open('$O/b4_$v.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
unset SPMM_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
