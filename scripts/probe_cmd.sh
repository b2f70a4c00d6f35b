cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/box_info.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp2 scripts/gather_probe2.cu
timeout 300 /tmp/gp2 22 65241671 > gpurun_out/gp2_22.txt 2>&1
timeout 400 /tmp/gp2 26 1060386521 > gpurun_out/gp2_26.txt 2>&1
