#!/bin/bash
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for rep in 1 2; do
for v in "X=0" "DFX_PAIR_STAGES=3" "DFX_PAIR_STAGES=3 DFX_BWD_CFG=3x1" "DFX_PAIR_STAGES=3 DFX_BWD_CFG=4x1" "DFX_PAIR_STAGES=3 DFX_BWD_CFG=3x2"; do
  env $v timeout 300 python bench.py $B > /tmp/k.log 2>&1
  echo "$v | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels"]["u_rowdot_tc"]["avg_us"], d["kernels"]["compose_bwd_dmag"]["avg_us"])' 2>&1 | tail -1)"
done; done
