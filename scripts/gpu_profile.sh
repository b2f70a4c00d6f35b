#!/bin/bash
# ncu evidence for round TAG: launch lists (per-kernel device time of a short bench run) and one
# `ncu --set full` capture of the compute kernel per workload, summarised on the box (text only).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
NCU=/usr/local/cuda/bin/ncu
BARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_${TAG}.csv python bench.py $BARGS > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config 2 $BARGS > /dev/null 2>&1
for spec in "1 auto rowsplit_c1" "2 auto merge_c2" "1 merge merge_c1" "0 auto rowsplit_c0"; do
  set -- $spec
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 1 -f \
    -o /tmp/prof_$3 python bench.py --config $1 --algo $2 $BARGS > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/prof_$3.ncu-rep --stalls > gpurun_out/ncu_$3_${TAG}.txt 2>&1
  python scripts/ncu_summary.py /tmp/prof_$3.ncu-rep --json >> gpurun_out/ncu_traffic_${TAG}.jsonl 2>/dev/null
done
[ -n "$KEEP_REP" ] && cp /tmp/prof_rowsplit_c1.ncu-rep gpurun_out/prof_rowsplit_c1_${TAG}.ncu-rep
ls -la gpurun_out
