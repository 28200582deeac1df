#!/bin/bash
# Norm plan strategy sweep (DFX_NORM_STRATEGY / DFX_NORM_SIDE overrides), norm alone and the
# inference / training bench lines.
mkdir -p gpurun_out; O=gpurun_out/strat.txt; : > $O
for b in 0 104; do
for v in "X=0" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=28" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=36" "DFX_NORM_STRATEGY=1 DFX_NORM_SIDE=20" "DFX_NORM_STRATEGY=2"; do
  env $v DFX_PLAN_PRINT=1 timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$v" >> $O 2>&1
done
done
for v in "X=0" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=28"; do
  env $v timeout 600 python bench.py --mode infer --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/strat_bench.log 2>&1
  echo "infer $v | $(tail -1 gpurun_out/strat_bench.log | cut -c1-150)" >> $O
done
for ns in 96 104 112 120; do
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/strat_bench.log 2>&1
  echo "train norm-sms $ns | $(tail -1 gpurun_out/strat_bench.log | cut -c1-150)" >> $O
done
grep -v "u plan" $O
