#!/bin/bash
# row split with 4-lane row groups (G = 4, NV = 4 float4 blocks at n = 64: 8 rows per warp, half the
# column-index / value broadcast loads) vs the default 8-lane groups, banded config 1, n = 64 / 128
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03c
mkdir -p $O
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], d['config'].get('algo'), 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  for v in default g4u4 g4u8; do
    L=""; [ $v != default ] && L="SPMM_LIB=build_variants/libspmm_$v.so"
    for n in 64 128; do
      env $L timeout 600 python bench.py --config 1 --n $n $BA > $O/c1_${v}_n${n}_$rep.json 2>$O/err_$v.txt; summ $O/c1_${v}_n${n}_$rep.json ${v}_n$n
    done
  done
done
