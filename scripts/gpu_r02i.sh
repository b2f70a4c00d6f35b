#!/bin/bash
# round 2: folded merge v2 + epilogue / split / iterative / fused-gather tests, timing
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02i
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -m gpu -x -q -k "worker or folded or queue or accumulate or execute_ex or split or iterative or fused or config0 or adversarial or identical" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
tail -30 $O/pytest_new.log
timeout 1200 python scripts/exp_fold.py 1,4,16 > $O/exp_fold.txt 2>&1; echo "exp rc=$?"
cat $O/exp_fold.txt
BA="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for c in 1 2 4; do
  timeout 600 python bench.py --config $c $BA > $O/b${c}.json 2> $O/b${c}.err
  echo "c$c: $(python -c "import json;d=json.load(open('$O/b${c}.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['config']['items_per_task'])" 2>&1 | tail -1)"
done
