#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/strat2.txt; : > $O
for v in "X=0" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=28" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=36"; do
  env $v DFX_V_GSTAT=1 timeout 120 python scripts/exp_norm_prof.py --budget 0 --iters 20 --tag "$v" >> $O 2>&1
done
for v in "X=0" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=28"; do
  env $v DFX_V_GSTAT=1 timeout 600 python bench.py --mode infer --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/strat_bench.log 2>&1
  echo "infer $v | $(tail -1 gpurun_out/strat_bench.log | cut -c1-150)" >> $O
done
cat $O
