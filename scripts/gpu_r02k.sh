#!/bin/bash
# round 2: per-shape folded tuning + values staged with their own TMA base: parity subset, sanitizers, timing
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02k
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "worker or folded or queue or misaligned or staging or config0 or adversarial or padding or accumulate or randomized" > $O/pytest_sub.log 2>&1; echo "rc=$?" >> $O/pytest_sub.log
tail -3 $O/pytest_sub.log
O=$O bash scripts/gpu_sanitize.sh
timeout 900 python scripts/exp_fold.py 1,2,4,8,16 > $O/exp_fold.txt 2>&1
cat $O/exp_fold.txt
BA="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for c in 1 2; do
  timeout 600 python bench.py --config $c $BA > $O/b${c}.json 2> $O/b${c}.err
  echo "c$c: $(python -c "import json;d=json.load(open('$O/b${c}.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
