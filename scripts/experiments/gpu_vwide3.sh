#!/bin/bash
# Inference step, V after U vs V wide on the side stream: 4 interleaved repeats each.
O=gpurun_out/vwide3.txt; : > $O
B="--mode infer --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0"
for rep in 1 2 3 4; do for v in "DFX_V_WIDE=0" "DFX_V_WIDE=1"; do
  env $v timeout 600 python bench.py $B > gpurun_out/vw_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/vw_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done; done
B="--mode train --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0"
for rep in 1 2; do for v in "DFX_V_WIDE=0" "DFX_V_WIDE=1"; do
  env $v timeout 600 python bench.py $B > gpurun_out/vw_bench.log 2>&1
  echo "train $v | $(tail -1 gpurun_out/vw_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done; done
cat $O
