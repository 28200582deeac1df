#!/bin/bash
# Pair-kernel K atoms per stage 2 vs 4 (DFX_PAIR_KA): live per-kernel times, the bench step, norm parity.
mkdir -p gpurun_out; O=gpurun_out/ka4.txt; : > $O
for b in 0 138; do
  for v in "DFX_PAIR_KA=2" "DFX_PAIR_KA=4" "DFX_PAIR_KA=2" "DFX_PAIR_KA=4"; do
    env $v DFX_PLAN_PRINT=1 timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$v" >> $O 2>&1
  done
done
B="--steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400"
for v in "DFX_PAIR_KA=2" "DFX_PAIR_KA=4" "DFX_PAIR_KA=2" "DFX_PAIR_KA=4"; do
  env $v timeout 600 python bench.py $B > gpurun_out/ka_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/ka_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "infer", d["variants"]["infer"]["value"], "U", d["kernels"]["u_rowdot_tc"]["avg_us"], d["roofline_step"])')" >> $O
done
DFX_PAIR_KA=4 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
    -o gpurun_out/ka4_ncu_tc_pair_rowdot python scripts/profile_module.py --steps 3 > /dev/null 2>&1
DFX_PAIR_KA=4 timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_vkernel.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ka4_tests.log 2>&1; echo "norm tests ka4 rc=$?" >> $O; tail -2 gpurun_out/ka4_tests.log >> $O
cat $O
