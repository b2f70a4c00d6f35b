#!/bin/bash
# round 2: e2e through the host-buffer call with a two-stream warm-up
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02t
mkdir -p $O
timeout 1500 python bench.py --no-extras --no-cpu-baseline --steps 5 --e2e-steps 4 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e'])"
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -12
