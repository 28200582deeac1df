#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/budget.txt; : > $O
for ns in 0 128 136 104; do
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/budget_bench.log 2>&1
  echo "train norm-sms $ns | $(tail -1 gpurun_out/budget_bench.log | cut -c1-150)" >> $O
done
for ns in 0 104; do
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --only norm --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/budget_bench.log 2>&1
  echo "norm-only norm-sms $ns | $(tail -1 gpurun_out/budget_bench.log | cut -c1-150)" >> $O
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --only compose --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/budget_bench.log 2>&1
  echo "compose-only norm-sms $ns | $(tail -1 gpurun_out/budget_bench.log | cut -c1-150)" >> $O
done
cat $O
