#!/bin/bash
# Round evidence on one B200: launch list + ncu full captures of the hot kernels.
# Usage (under gpurun): bash scripts/round_profile.sh r01
R=${1:-r01}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
for k in tc_pair_rowdot compose_fwd_vec compose_bwd_serial tc_rowdot; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${R}_ncu_$k python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
done
# the W.A^T GEMM as planned under the pipelined bench's SM budget (full r per pair)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
    -o gpurun_out/${R}_ncu_tc_pair_rowdot_budget104 python scripts/profile_module.py --steps 3 --budget 104 > /dev/null 2>&1
# the fused LoRA-up GEMM + compose epilogue
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lora_compose -s 2 -c 1 \
    -o gpurun_out/${R}_ncu_lora_compose python scripts/exp_kernels.py --what lora_fused --iters 1 > /dev/null 2>&1
ls gpurun_out | grep $R
# fp32 weights on the tensor cores (3xTF32, BASELINE configs[0])
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_rowdot -s 1 -c 1 \
    -o gpurun_out/${R}_ncu_tc_rowdot_tf32x3_c1 python scripts/profile_module.py --config c1 --steps 2 > /dev/null 2>&1
