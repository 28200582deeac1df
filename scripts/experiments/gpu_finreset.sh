#!/bin/bash
B="--steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400"
for rep in 1 2; do for v in 0 1; do
  DFX_FIN_RESET=$v timeout 300 python bench.py $B > /tmp/f.log 2>&1
  echo "reset $v | $(tail -1 /tmp/f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"])')"
done; done
