#!/bin/bash
mkdir -p gpurun_out
DFX_V_GSTAT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_pair_gstat" -s 1 -c 1 \
    -o gpurun_out/c3_ncu_gstat python scripts/profile_module.py --config c3 --steps 3 > gpurun_out/c3_ncu.log 2>&1
ls gpurun_out | grep c3_ncu
