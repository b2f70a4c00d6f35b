#!/bin/bash
# merge at 6 CTAs per SM (48 warps, 40 registers; the spills sit outside the gather loop) vs 5 (40 warps)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03j
mkdir -p $O
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], d['config'].get('algo'), 'step %.4f ms'%d['ms_per_step'], 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  timeout 600 python bench.py --config 2 $BA > $O/c2_mb5_$rep.json 2>/dev/null; summ $O/c2_mb5_$rep.json c2_mb5
  SPMM_LIB=build_variants/libspmm_mb6.so timeout 600 python bench.py --config 2 $BA > $O/c2_mb6_$rep.json 2>/dev/null; summ $O/c2_mb6_$rep.json c2_mb6
done
for rep in 1 2; do
  timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_mb5_$rep.json 2>/dev/null; summ $O/c4_mb5_$rep.json c4_mb5
  SPMM_LIB=build_variants/libspmm_mb6.so timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_mb6_$rep.json 2>/dev/null; summ $O/c4_mb6_$rep.json c4_mb6
done
timeout 600 python scripts/exp_small_n.py 32,64 > $O/small_mb5.txt 2>&1
SPMM_LIB=build_variants/libspmm_mb6.so timeout 600 python scripts/exp_small_n.py 32,64 > $O/small_mb6.txt 2>&1
cat $O/small_mb5.txt $O/small_mb6.txt
