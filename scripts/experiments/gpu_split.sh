#!/bin/bash
B="--steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 2"
timeout 300 python bench.py $B > /tmp/s.log 2>&1; echo "base train | $(tail -1 /tmp/s.log | cut -c 60-100)"
for as in 12 20 28 40 60; do
  timeout 300 python bench.py $B --split-adapter 1 --adapter-sms $as > /tmp/s.log 2>&1
  echo "split train adapter-sms $as rc=$? | $(tail -1 /tmp/s.log | cut -c 60-100)"
done
timeout 300 python bench.py $B --mode infer > /tmp/s.log 2>&1; echo "base infer | $(tail -1 /tmp/s.log | cut -c 60-100)"
for as in 20 28 40 60; do
  timeout 300 python bench.py $B --mode infer --split-adapter 1 --adapter-sms $as > /tmp/s.log 2>&1
  echo "split infer adapter-sms $as rc=$? | $(tail -1 /tmp/s.log | cut -c 60-100)"
done
