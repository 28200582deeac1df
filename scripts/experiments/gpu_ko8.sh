#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 $EXTRA > /dev/null 2>&1; }
for d in 1024 4096; do for ka in 1 2; do
  EXTRA="--d-out $d" run s_all_d${d}_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_s_all.so
done; done
