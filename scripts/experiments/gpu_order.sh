#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/order.txt; : > $O
B="--steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0"
for rep in 1 2; do
for v in "--capture-order module" "--capture-order norm-first" "--nbuf 3" "--nbuf 6" "--norm-sms 144 --capture-order norm-first"; do
  timeout 300 python bench.py $B $v > gpurun_out/order_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/order_bench.log | cut -c1-110)" >> $O
done
done
for v in "--mode infer --capture-order norm-first" "--mode infer --capture-order module" "--mode infer --norm-sms 140"; do
  timeout 300 python bench.py $B $v > gpurun_out/order_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/order_bench.log | cut -c1-110)" >> $O
done
cat $O
