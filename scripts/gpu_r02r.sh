#!/bin/bash
# round 2: host-buffer C-ABI call (parity + e2e), ncu traffic refresh for this build, default bench line
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02r
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py tests/test_c_abi_program.py -m gpu -x -q -k "multiply_host or graph or bench or cuda_arm or torchrun or abi" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python scripts/ncu_traffic.py $O/ncu_traffic.json > $O/ncu_traffic.log 2>&1; echo "ncu_traffic rc=$?"
cp $O/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ncu']['same_build'], d['e2e'])"
