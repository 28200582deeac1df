#!/bin/bash
B="--no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0 --warmup 20"
for v in "--steps 20" "--steps 40" "--steps 200" "--steps 200 --pipeline 20" "--steps 2000" "--steps 2000 --pipeline 20" "--steps 20"; do
  timeout 300 python bench.py $B $v > /tmp/p.log 2>&1
  echo "$v | $(tail -1 /tmp/p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"]["pipeline"][:22], d["clocks"])')"
done
