#!/bin/bash
# training-step norm SM budget re-check on the final build (400-step runs, two repeats)
mkdir -p gpurun_out; O=gpurun_out/budget3.txt; : > $O
for rep in 1 2; do for ns in 134 136 138 140 142 146; do
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/b3.log 2>&1
  echo "train norm-sms $ns | $(tail -1 gpurun_out/b3.log | cut -c60-100)" >> $O
done; done
cat $O
