#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lora_compose -s 2 -c 1 -o gpurun_out/ncu_lora5 python scripts/exp_kernels.py --what lora_fused --iters 1 > gpurun_out/ncu_lora.log 2>&1
