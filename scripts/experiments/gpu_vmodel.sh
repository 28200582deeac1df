#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for cfg in c2 c3 c4r64 c4r128 c4r512 c4r1024; do for mode in train infer; do
  DFX_PLAN_PRINT=1 timeout 300 python bench.py $B --config $cfg --mode $mode > /tmp/k.log 2>&1
  echo "$cfg $mode | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("norm_sm_budget"))' 2>&1 | tail -1) | $(grep 'u plan' /tmp/k.log | sort | uniq -c | sort -rn | head -1 | cut -c1-130)"
done; done
