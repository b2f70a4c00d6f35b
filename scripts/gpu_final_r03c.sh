#!/bin/bash
# final evidence of round 2 (session 3), part C, with the final build (k_partition 16 rows per thread):
# full GPU suite, smoke, ncu traffic of the bench's kernels (profiles/ncu_traffic.json, with the source
# hash), launch lists, bench lines, memcheck of the merge path, small-n AUTO table
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/final3c
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
sha256sum paper_1803_08601_b200/libspmm.so | cut -c1-16 > $O/lib_sha16.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python scripts/ncu_traffic.py $O/ncu_traffic.json > $O/ncu_traffic.log 2>&1; echo "ncu_traffic rc=$?"
cp $O/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
BARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
for c in 1 2 4; do
  timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:k_tile|k_merge_|k_partition|k_fixup|k_max_row|k_tiled" \
    --csv --log-file $O/launches_c$c.csv \
    python bench.py --config $c $BARGS > /dev/null 2>&1; echo "launches c$c rc=$?"
done
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --config 1 --no-extras > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?"
timeout 900 python bench.py --config 2 --no-extras > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 1 --n 128 --no-extras --no-e2e > $O/bench_c1_n128.json 2> $O/bench_c1_n128.err; echo "bench c1 n128 rc=$?"
cut -c1-400 $O/bench_default.json
timeout 900 python scripts/exp_small_n.py 1,4,16,64 > $O/small_n.txt 2>&1; cat $O/small_n.txt
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "merge_partitions or partition_kernel or (merge_worker_parity and rmat12 and (f32_plus_times or i32_min_plus) and (1- or 16-)) or merge_task_queue or (adversarial and merge and (giant or rmat12 or many_empty or leading))" > $O/sanitize_memcheck_merge.log 2>&1; echo "memcheck rc=$?" >> $O/sanitize_memcheck_merge.log
tail -3 $O/sanitize_memcheck_merge.log
