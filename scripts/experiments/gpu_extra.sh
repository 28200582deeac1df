#!/bin/bash
mkdir -p gpurun_out
for mode in train infer; do
  timeout 600 python bench.py --config c5 --mode $mode --steps 3 --warmup 3 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline > gpurun_out/r02_c5_$mode.log 2>&1; echo "c5 $mode rc=$? $(tail -1 gpurun_out/r02_c5_$mode.log | cut -c1-160)"
done
for ar in dfx nccl; do
  timeout 600 python bench.py --mode dsplit --allreduce $ar --steps 20 --warmup 5 > gpurun_out/r02_dsplit_$ar.log 2>&1; echo "dsplit $ar rc=$? $(tail -1 gpurun_out/r02_dsplit_$ar.log | cut -c1-300)"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"compose_bwd_serial" -s 0 -c 1 \
    -o gpurun_out/r02h_ncu_compose_bwd_partitioned python scripts/profile_module.py --steps 2 --bwd --budget 138 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"compose_fwd_vec" -s 0 -c 1 \
    -o gpurun_out/r02h_ncu_compose_fwd python scripts/profile_module.py --steps 2 --bwd > /dev/null 2>&1
ls gpurun_out | grep r02h
