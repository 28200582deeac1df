#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:tc_pair_rowdot --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
run base_ka1 DFX_PAIR_KA=1
run koall_ka1 DFX_PAIR_KA=1 DFX_LIB=variants/libdfx_ko_all.so
run koall_ka2 DFX_PAIR_KA=2 DFX_LIB=variants/libdfx_ko_all.so
run koallc_ka1 DFX_PAIR_KA=1 DFX_LIB=variants/libdfx_ko_allc.so
run koallc_ka2 DFX_PAIR_KA=2 DFX_LIB=variants/libdfx_ko_allc.so
run komma_ka1 DFX_PAIR_KA=1 DFX_LIB=variants/libdfx_ko_mma.so
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_22276_b200/csrc/kernels tma_tensor_micro.cu -o tma_tensor_micro -lcuda && ./tma_tensor_micro) > gpurun_out/ko/tma_micro.txt 2>&1
ls gpurun_out/ko
