#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
for v in ko_mma ko_chain ko_both ko_epi ko_mce; do run t3_$v DFX_LIB=variants/libdfx_$v.so; done
