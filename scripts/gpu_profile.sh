#!/bin/bash
# ncu evidence: launch list (per-kernel device time of one bench run) + one full capture per kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
NCU=/usr/local/cuda/bin/ncu
BARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_${TAG}.csv python bench.py $BARGS > gpurun_out/ncu_launch_c1.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config 2 $BARGS > gpurun_out/ncu_launch_c2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 1 -f -o gpurun_out/prof_rowsplit_c1_${TAG} python bench.py $BARGS > gpurun_out/ncu_full_c1.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 1 -f -o gpurun_out/prof_merge_c2_${TAG} python bench.py --config 2 $BARGS > gpurun_out/ncu_full_c2.log 2>&1
ls -la gpurun_out/
