#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:tc_pair_rowdot --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
run base2 X=0
run sleep256 DFX_LIB=variants/libdfx_sleep256.so
run sleep1k DFX_LIB=variants/libdfx_sleep1k.so
run koall_sleep DFX_LIB=variants/libdfx_koall_sleep.so
run koall2 DFX_LIB=variants/libdfx_ko_all.so
for v in X=0 DFX_LIB=variants/libdfx_sleep1k.so; do
  env $v timeout 120 python scripts/exp_norm_prof.py --budget 0 --iters 20 --tag "$v" >> gpurun_out/ko/sleep_live.txt 2>&1
done
ls gpurun_out/ko
