#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for cfg in c3 c4r512 c4r1024 c4r64; do
  for ns in 0 104 120; do
    timeout 300 python bench.py $B --config $cfg --norm-sms $ns > /tmp/k.log 2>&1
    echo "$cfg train norm-sms $ns | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])' 2>&1 | tail -1)"
  done
done
