#!/bin/bash
# V on the side stream with an all-SM grid (DFX_V_WIDE=1) vs V after U, after the V latency work.
O=gpurun_out/vwide2.txt; : > $O
for b in 0 138; do for v in "DFX_V_WIDE=0" "DFX_V_WIDE=1"; do
  env $v timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$v" >> $O 2>&1
done; done
B="--steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400"
for v in "DFX_V_WIDE=0" "DFX_V_WIDE=1" "DFX_V_WIDE=0" "DFX_V_WIDE=1"; do
  env $v timeout 600 python bench.py $B > gpurun_out/vw_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/vw_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], "infer", d["variants"]["infer"]["value"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done
cat $O
