#!/bin/bash
# Round evidence on one B200: full GPU tests, smoke, the driver's bench commands, launch list and
# ncu full captures of the norm kernels.  Usage: bash scripts/gpu_round.sh TAG
R=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${R}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${R}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${R}_smoke.log
timeout 900 python bench.py > gpurun_out/${R}_bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${R}_bench_default.log | cut -c1-300
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench_s20.log 2>&1; echo "bench s20 rc=$?"; tail -1 gpurun_out/${R}_bench_s20.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${R}_bench_ref.log | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_pair_rowdot|tc_pair_gstat|tc_rowdot|gram_reduce" -s 0 -c 4 \
    -o gpurun_out/${R}_ncu_norm python scripts/profile_module.py --steps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
    -o gpurun_out/${R}_ncu_tc_pair_rowdot_budget104 python scripts/profile_module.py --steps 3 --budget 104 > /dev/null 2>&1
# the composes and the fused LoRA-up + compose kernel, and the bench's own launch list
for k in compose_fwd_vec compose_bwd_serial; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${R}_ncu_$k python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lora_compose -s 2 -c 1 \
    -o gpurun_out/${R}_ncu_lora_compose python scripts/exp_kernels.py --what lora_fused --iters 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_bench_launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline \
    --e2e-steps 1 --lora-steps 2 --variant-steps 40 > /dev/null 2>&1
ls gpurun_out | grep $R
