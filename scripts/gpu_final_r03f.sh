#!/bin/bash
# final evidence of round 2 (session 3), part F, with the final build (+ float2 folded slots, L = 6 float4 narrow slots):
# full GPU suite, smoke, ncu traffic of the bench's kernels (profiles/ncu_traffic.json, with the source
# hash), launch lists, bench lines, small-n AUTO table, BASELINE configs[3] sweep, scaling emulation
# (compute-sanitizer is closed on this pool)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/final3f
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
timeout 3000 python scripts/sweep_config4.py --out $O/config3 > $O/config3.log 2>&1; echo "config3 rc=$?"
tail -8 $O/config3.log
timeout 2400 python scripts/scaling_emulation.py --config 4 --out $O/scaling_emulation_config4 > $O/scaling4.log 2>&1; echo "scaling rc=$?"
tail -7 $O/scaling4.log
