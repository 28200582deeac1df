#!/bin/bash
# Round evidence on one B200: config sweep + launch list + ncu full captures of the hot kernels.
# Usage (under gpurun): bash scripts/round_profile.sh r01
R=${1:-r01}
mkdir -p gpurun_out
for cfg in c1 c3 c4r64 c4r128 c4r512 c4r1024; do
  timeout 300 python bench.py --config $cfg --steps 300 --e2e-steps 0 --no-cpu-baseline \
      > gpurun_out/${R}_cfg_$cfg.json 2> gpurun_out/${R}_cfg_$cfg.err || echo "cfg $cfg failed"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
for k in tc_pair_rowdot compose_fwd_vec compose_bwd_serial; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${R}_ncu_$k python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
done
ls gpurun_out | grep $R
