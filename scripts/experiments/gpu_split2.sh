#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for mode in train infer; do
  timeout 300 python bench.py $B --mode $mode > /tmp/s.log 2>&1; echo "$mode base | $(tail -1 /tmp/s.log | cut -c 60-100)"
  for as in 12 20 28 40; do
    timeout 300 python bench.py $B --mode $mode --split-adapter 1 --adapter-sms $as > /tmp/s.log 2>&1
    echo "$mode split after adapter-sms $as rc=$? | $(tail -1 /tmp/s.log | cut -c 60-100)"
  done
done
