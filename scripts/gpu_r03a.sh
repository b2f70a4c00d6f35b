#!/bin/bash
# re-entry check: full GPU suite, smoke, default bench line and heads 1 / 2
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python bench.py --config 1 --no-extras --no-e2e --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?"
timeout 900 python bench.py --config 2 --no-extras --no-e2e --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
python -c "
import json
for c in (1,2):
    d=json.load(open('$O/bench_c%d.json'%c)); r=d['roofline']; print(c, d['ms_per_step'], r['avg_launch_ms'], r['frac'])"
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
