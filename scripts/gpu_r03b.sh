#!/bin/bash
# round 2 (session 3): LDS broadcast probe; rolling merge pipeline (MW_ROLL) and rotated row walk (RS_ROT)
# A/B against the previous kernels; merge / row-split parity subset with the new default
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03b
mkdir -p $O
./scripts/lds_bcast_probe > $O/lds_bcast_probe.txt 2>&1; cat $O/lds_bcast_probe.txt
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']; print(sys.argv[2], d['config'].get('algo'), 'step %.4f ms'%d['ms_per_step'], 'kernel %.4f ms'%r['avg_launch_ms'], 'frac %.4f'%r['frac'])" $1 $2; }
for rep in 1 2; do
  timeout 600 python bench.py --config 1 $BA > $O/c1_rot_$rep.json 2>/dev/null; summ $O/c1_rot_$rep.json c1_rot
  SPMM_LIB=build_variants/libspmm_norot.so timeout 600 python bench.py --config 1 $BA > $O/c1_norot_$rep.json 2>/dev/null; summ $O/c1_norot_$rep.json c1_norot
  timeout 600 python bench.py --config 2 $BA > $O/c2_roll_$rep.json 2>/dev/null; summ $O/c2_roll_$rep.json c2_roll
  SPMM_LIB=build_variants/libspmm_noroll.so timeout 600 python bench.py --config 2 $BA > $O/c2_noroll_$rep.json 2>/dev/null; summ $O/c2_noroll_$rep.json c2_noroll
done
timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_roll.json 2>/dev/null; summ $O/c4_roll.json c4_roll
SPMM_LIB=build_variants/libspmm_noroll.so timeout 900 python bench.py --config 4 $BA --steps 10 > $O/c4_noroll.json 2>/dev/null; summ $O/c4_noroll.json c4_noroll
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config0 or adversarial or merge_worker or every_row or b_staging or randomized or misaligned or bit_identical or folded" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_subset.log
