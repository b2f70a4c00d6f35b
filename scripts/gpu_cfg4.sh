#!/bin/bash
# BASELINE configs[4] (R-MAT scale 26, n=64) on one B200: generation + AUTO kernel + both partitions
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/cfg4_mem.txt 2>&1
( time timeout 1200 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ) > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -n 5 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
