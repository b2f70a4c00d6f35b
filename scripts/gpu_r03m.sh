#!/bin/bash
# default bench line again on another box (the e2e leg is bound by the host link, which varies by box)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03m
mkdir -p $O
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv | tee $O/pcie.txt
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'], d['config1']['e2e'] if 'e2e' in d['config1'] else '')"
