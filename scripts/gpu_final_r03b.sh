#!/bin/bash
# final evidence of round 2 (session 3), part B, same build: compute-sanitizer, BASELINE configs[3]
# (n sweep x 27 matrices, AUTO accuracy), scaling emulation of configs[4]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/final3
mkdir -p $O
sha256sum paper_1803_08601_b200/libspmm.so | cut -c1-16 > $O/lib_sha16_b.txt
# compute-sanitizer is closed on this pool (rc 86); the sanitizer evidence is profiles/r02_sanitize_*.log
timeout 3000 python scripts/ncu_traffic.py $O/ncu_traffic_b.json > $O/ncu_traffic_b.log 2>&1; echo "ncu_traffic b rc=$?"
timeout 3000 python scripts/sweep_config4.py --out $O/config3 > $O/config3.log 2>&1; echo "config3 rc=$?"
tail -8 $O/config3.log
timeout 2400 python scripts/scaling_emulation.py --config 4 --out $O/scaling_emulation_config4 > $O/scaling4.log 2>&1; echo "scaling rc=$?"
tail -7 $O/scaling4.log
