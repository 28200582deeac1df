#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 $EXTRA > /dev/null 2>&1; }
for ka in 1 2; do
  run s_split_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_s_split.so
  run b_split_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_b_split.so
done
EXTRA="--d-out 1024" run s_split_d1024 DFX_LIB=variants/libdfx_s_split.so
