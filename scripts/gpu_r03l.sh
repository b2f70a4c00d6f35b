#!/bin/bash
# k_partition with coalesced, shared-memory staged row offsets: parity subset, launch times
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03l
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "partition or merge_worker or folded or task_queue or adversarial or config0 or rmat26 or every_row" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
BARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
for c in 2 4; do
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:k_partition" --csv --log-file $O/launches_c$c.csv python bench.py --config $c $BARGS > /dev/null 2>&1
grep -h "k_partition" $O/launches_c$c.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -3
done
