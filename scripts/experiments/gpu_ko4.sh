#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:tc_pair_rowdot --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
for ka in 1 2; do
run s_c_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_ko_allc.so
run s_fwd_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_s_fwd.so
run s_fwd_tmem_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_s_fwd_tmem.so
done
(cd tools && ./tma_tensor_micro > /dev/null 2>&1; timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:pair_kernel --csv --log-file ../gpurun_out/ko/replica.csv ./tma_tensor_micro > /dev/null 2>&1)
ls gpurun_out/ko
