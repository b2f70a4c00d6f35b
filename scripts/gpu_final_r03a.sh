#!/bin/bash
# final evidence of round 2 (session 3), part A, with the final build: ncu traffic of the bench's kernels
# (profiles/ncu_traffic.json), launch lists, ncu --set full summaries, the bench lines (default = configs[4]
# + heads 1 / 2, the reference arm), the full GPU suite and smoke.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/final3
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
sha256sum paper_1803_08601_b200/libspmm.so | cut -c1-16 > $O/lib_sha16.txt
timeout 3000 python scripts/ncu_traffic.py $O/ncu_traffic.json > $O/ncu_traffic.log 2>&1; echo "ncu_traffic rc=$?"
cp $O/ncu_traffic.json profiles/ncu_traffic.json 2>/dev/null
BARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
for c in 1 2 4; do
  timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:k_tile|k_merge_|k_partition|k_fixup|k_max_row|k_tiled" \
    --csv --log-file $O/launches_c$c.csv \
    python bench.py --config $c $BARGS > /dev/null 2>&1; echo "launches c$c rc=$?"
done
for spec in "1 k_tile< rowsplit_c1" "2 k_merge_w< merge_c2"; do
  set -- $spec
  timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s 2 -c 1 -f \
    -o $O/prof_$3 python bench.py --config $1 $BARGS > /dev/null 2>&1
  python scripts/ncu_summary.py $O/prof_$3.ncu-rep --stalls > $O/ncu_$3.txt 2>&1; echo "full $3 done"
done
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --config 1 --no-extras > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?"
timeout 900 python bench.py --config 2 --no-extras > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 1 --n 128 --no-extras --no-e2e > $O/bench_c1_n128.json 2> $O/bench_c1_n128.err; echo "bench c1 n128 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench ref rc=$?"
cut -c1-600 $O/bench_default.json
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
