#!/bin/bash
for ns in 80 96 104 112 120; do
  timeout 600 python bench.py --config c5 --mode train --steps 3 --warmup 3 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline --norm-sms $ns > /tmp/c5.log 2>&1; echo "c5 train norm-sms $ns rc=$? | $(tail -1 /tmp/c5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done
for ns in 0 104; do
  timeout 600 python bench.py --config c5 --mode infer --steps 3 --warmup 3 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline --norm-sms $ns > /tmp/c5.log 2>&1; echo "c5 infer norm-sms $ns rc=$? | $(tail -1 /tmp/c5.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done
