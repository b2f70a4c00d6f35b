#!/bin/bash
# round 2: host-buffer call with 1-D copies: e2e timing, multiply_host parity, ncu traffic refresh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multiply_host" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 3000 python scripts/ncu_traffic.py $O/ncu_traffic.json > $O/ncu_traffic.log 2>&1; echo "ncu_traffic rc=$?"
cp $O/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ncu']['same_build'], d['e2e'])"
