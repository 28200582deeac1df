#!/bin/bash
mkdir -p gpurun_out
DFX_V_GSTAT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_pair_gstat" -s 1 -c 1 \
    -o gpurun_out/gs_ncu_gstat python scripts/profile_module.py --steps 3 > gpurun_out/gs_ncu.log 2>&1
DFX_V_GSTAT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/gs_launches.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1
ls gpurun_out | grep gs_
