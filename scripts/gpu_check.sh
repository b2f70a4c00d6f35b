#!/bin/bash
# quick GPU round: smoke, gpu tests, bench lines. Outputs under gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
[ -z "$SKIP_TESTS" ] && timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config 2 --algo rowsplit --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_rs.json 2> gpurun_out/bench_c2_rs.err
timeout 600 python bench.py --config 1 --algo merge --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_merge.json 2> gpurun_out/bench_c1_merge.err
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/smoke.log; cat gpurun_out/bench_*.json; for f in gpurun_out/bench_*.err; do tail -n 3 $f; done
