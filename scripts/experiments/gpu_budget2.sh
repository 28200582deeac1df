#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/budget2.txt; : > $O
for ns in 132 136 140 144 148 120 112; do
  DFX_PLAN_PRINT=1 timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/budget_bench.log 2>&1
  echo "train norm-sms $ns | $(grep 'u plan' gpurun_out/budget_bench.log | sort | uniq -c | head -3) | $(tail -1 gpurun_out/budget_bench.log | cut -c1-120)" >> $O
done
cat $O
