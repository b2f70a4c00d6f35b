#!/bin/bash
# round 2: pipelined e2e + CUDA-graph capture test + smoke; the default bench line
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02q
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -m gpu -x -q -k "graph or bench or cuda_arm or torchrun" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'])"
