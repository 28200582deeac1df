#!/bin/bash
# ncu full captures of the U GEMM and the d_mag backward + mma microbenchmark (analysis)
mkdir -p gpurun_out
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_22276_b200/csrc/kernels mma_micro.cu -o mma_micro -lcuda && ./mma_micro) > gpurun_out/mma_micro.txt 2>&1
for k in ${@:-tc_pair_rowdot compose_bwd_serial}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/ncu_$k python scripts/profile_module.py --steps 3 --bwd > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
