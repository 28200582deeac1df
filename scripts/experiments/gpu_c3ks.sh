#!/bin/bash
B="--config c3 --steps 40 --warmup 10 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 40 --e2e-steps 0"
for v in "X=0" "DFX_U_KS=2 DFX_U_NH=2" "DFX_U_KS=4 DFX_U_NH=2" "DFX_U_KS=2 DFX_U_NH=1" "DFX_U_KS=1 DFX_U_NH=1"; do
  env $v DFX_PLAN_PRINT=1 timeout 120 python scripts/exp_norm_prof.py --config c3 --budget 0 --iters 10 --tag "$v" 2>&1 | grep -v "u plan" 
  env $v timeout 300 python bench.py $B > /tmp/k.log 2>&1
  echo "$v | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"])' 2>&1 | tail -1)"
done
DFX_U_KS=2 DFX_U_NH=2 timeout 600 python -m pytest tests/test_gpu_norm.py -q -k "c3_four_chunks" -p no:cacheprovider 2>&1 | tail -1
