#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/wide.txt; : > $O
for v in "X=0" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=12 DFX_V_WIDE=1" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20 DFX_V_WIDE=1" "DFX_NORM_STRATEGY=0 DFX_NORM_SIDE=20 DFX_V_WIDE=1 DFX_V_GSTAT=0"; do
  env $v timeout 120 python scripts/exp_norm_prof.py --budget 0 --iters 20 --tag "$v" >> $O 2>&1
  env $v timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/wide_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/wide_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], d["ms_per_step"], "infer", d["variants"]["infer"]["value"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done
cat $O
