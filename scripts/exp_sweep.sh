#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair -s 1 -c 1 -o gpurun_out/ncu_u_nh2 python scripts/profile_module.py --budget 80 --steps 2 > gpurun_out/ncu_u.log 2>&1
