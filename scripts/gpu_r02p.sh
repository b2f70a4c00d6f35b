#!/bin/bash
# round 2: row pairs (plan-time table) -- parity + banded timing with pairs on / off
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02p
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "row_pairs or tiled or config0 or staging or misaligned" > $O/pytest_pairs.log 2>&1; echo "rc=$?" >> $O/pytest_pairs.log
tail -15 $O/pytest_pairs.log
BA="--config 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for rp in off on; do
  timeout 600 python bench.py $BA --row-pairs $rp > $O/b1_$rp.json 2> $O/b1_$rp.err
  echo "c1 pairs $rp: $(python -c "import json;d=json.load(open('$O/b1_$rp.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
for n in 16 32 128; do for rp in off on; do
  timeout 600 python bench.py $BA --n $n --row-pairs $rp > $O/b1_n${n}_$rp.json 2> $O/b1_n${n}_$rp.err
  echo "c1 n=$n pairs $rp: $(python -c "import json;d=json.load(open('$O/b1_n${n}_$rp.json'));print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)"
done; done
