#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for rep in 1 2; do
for ns in 134 136 137 138 139 140; do
  DFX_PLAN_PRINT=1 timeout 300 python bench.py $B --norm-sms $ns > /tmp/k.log 2>&1
  echo "$ns | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])' 2>&1 | tail -1) | $(grep 'u plan' /tmp/k.log | grep "sms $ns" | sort -u | cut -c1-120 | head -1)"
done; done
