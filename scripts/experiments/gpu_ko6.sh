#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 $FILLARG > /dev/null 2>&1; }
for f in zeros bits randn; do
  FILLARG="--fill $f" run fill_${f}_skel DFX_LIB=variants/libdfx_ko_allc.so
  FILLARG="--fill $f" run fill_${f}_base X=0
done
