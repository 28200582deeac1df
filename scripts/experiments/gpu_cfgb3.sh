#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for ns in 112 116 120 124 128 136; do
  DFX_PLAN_PRINT=1 timeout 300 python bench.py $B --config c3 --norm-sms $ns > /tmp/k.log 2>&1
  echo "c3 train norm-sms $ns | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])' 2>&1 | tail -1) | $(grep 'u plan' /tmp/k.log | grep "sms $ns" | sort -u | head -1 | cut -c1-110)"
done
for ns in 0 120; do
  timeout 300 python bench.py $B --config c3 --mode infer --norm-sms $ns > /tmp/k.log 2>&1
  echo "c3 infer norm-sms $ns | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])' 2>&1 | tail -1)"
done
