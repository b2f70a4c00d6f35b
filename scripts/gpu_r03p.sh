#!/bin/bash
# merge kernels with a shared-memory carveout preference of 0% / 25% (the rest of L1 caches B rows) vs default
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03p
mkdir -p $O
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], 'step %.4f ms'%d['ms_per_step'], 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  timeout 600 python bench.py --config 2 $BA > $O/c2_def_$rep.json 2>/dev/null; summ $O/c2_def_$rep.json c2_default
  for v in co0 co25; do SPMM_LIB=build_variants/libspmm_$v.so timeout 600 python bench.py --config 2 $BA > $O/c2_${v}_$rep.json 2>/dev/null; summ $O/c2_${v}_$rep.json c2_$v; done
done
timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_def.json 2>/dev/null; summ $O/c4_def.json c4_default
SPMM_LIB=build_variants/libspmm_co0.so timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_co0.json 2>/dev/null; summ $O/c4_co0.json c4_co0
timeout 600 python scripts/exp_small_n.py 1,16,64 > $O/small_def.txt 2>&1; SPMM_LIB=build_variants/libspmm_co0.so timeout 600 python scripts/exp_small_n.py 1,16,64 > $O/small_co0.txt 2>&1; cat $O/small_def.txt $O/small_co0.txt
