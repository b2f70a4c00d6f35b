#!/bin/bash
# fixup: runs of carries resolved 32 at a time (ballot); parity subset, config 2 step, launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r03h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -m gpu -q -x -k "partition or merge or folded or task_queue or bit_identical or accumulate or adversarial or randomized or misaligned or config0 or fused or iterative" > $O/pytest_subset.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.log
BA="--no-extras --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
for rep in 1 2; do
timeout 600 python bench.py --config 2 $BA > $O/c2_$rep.json 2>/dev/null
python -c "import json;d=json.load(open('$O/c2_$rep.json'));r=d['roofline'];print('c2 step', d['ms_per_step'], 'kernel', r['avg_launch_ms'], r['frac'])"
done
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat22_n64.csv python scripts/run_one.py rmat22 64 merge > /dev/null 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat20_n1.csv python scripts/run_one.py rmat20 1 merge folded > /dev/null 2>&1
python - <<'PY'
import csv
for f in ['gpurun_out/r03h/launches_rmat20_n1.csv','gpurun_out/r03h/launches_rmat22_n64.csv']:
    rows=list(csv.reader(open(f)))
    for i,r in enumerate(rows):
        if 'Kernel Name' in r: hdr=r; start=i+1; break
    ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value')
    print(f, [ (r[ik][6:18], r[iv]) for r in rows[start:] if 'spmm::' in r[ik]][:6])
PY
