#!/bin/bash
# round 2: merge-kernel variants on R-MAT 22/26, HBM random-gather ceiling probe, 1-D vs 2-D partition ablation,
# ncu DRAM bytes of k_merge_w on R-MAT 26
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/r02d
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp3 scripts/gather_probe3.cu
timeout 600 /tmp/gp3 26 268435456 > $O/gp3_26.txt 2>&1
timeout 300 /tmp/gp3 22 65241671 > $O/gp3_22.txt 2>&1
cat $O/gp3_26.txt $O/gp3_22.txt
BA="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for v in default noalloc cg u16mb4 mb6; do
  if [ $v = default ]; then export SPMM_LIB=$PWD/paper_1803_08601_b200/libspmm.so; else export SPMM_LIB=$PWD/build_variants/lib_$v.so; fi
  for c in 2 4; do
    timeout 600 python bench.py --config $c $BA > $O/b${c}_$v.json 2> $O/b${c}_$v.err
    echo "$v c$c: $(python -c "import json;d=json.load(open('$O/b${c}_$v.json'));print(d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" 2>&1 | tail -1)"
  done
done
unset SPMM_LIB
timeout 1200 python scripts/ablation_partition.py --big --out $O/ablation_partition > $O/ablation.txt 2>&1; echo "ablation rc=$?"
cat $O/ablation.txt
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct \
  --clock-control none -k regex:k_merge_w -s 1 -c 1 --csv --log-file $O/ncu_c4_dram.csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "ncu rc=$?"
cat $O/ncu_c4_dram.csv | tail -8
