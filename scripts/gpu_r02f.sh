#!/bin/bash
# round 2: lane-folded merge parity + worker/task-queue experiments
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02f
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "worker or folded or queue or config0 or adversarial or partitions or identical" > $O/pytest_fold.log 2>&1; echo "rc=$?" >> $O/pytest_fold.log
tail -15 $O/pytest_fold.log
timeout 1200 python scripts/exp_fold.py > $O/exp_fold.txt 2>&1; echo "exp rc=$?"
cat $O/exp_fold.txt
BA="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for c in 2 4; do for t in 1 2 4 8; do
  timeout 600 python bench.py --config $c --tasks-per-warp $t $BA > $O/b${c}_t$t.json 2> $O/b${c}_t$t.err
  echo "c$c tpw$t: $(python -c "import json;d=json.load(open('$O/b${c}_t$t.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done; done
