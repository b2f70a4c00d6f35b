#!/bin/bash
# round evidence: ncu launch lists + full captures (scripts/gpu_profile.sh) and the bench lines of
# configs 1 (default), 2 and 4
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01} bash scripts/gpu_profile.sh > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_final_c1.json 2> gpurun_out/bench_final_c1.err
timeout 900 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench_final_c2.json 2> gpurun_out/bench_final_c2.err
timeout 1200 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_final_c4.json 2> gpurun_out/bench_final_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
ls gpurun_out/*r01* ; cut -c1-300 gpurun_out/bench_final_*.json; tail -n 3 gpurun_out/bench_final_*.err
