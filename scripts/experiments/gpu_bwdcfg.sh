#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/bwdcfg.txt; : > $O
B="--steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0"
for rep in 1 2; do
for c in 6x2 4x2 3x2 6x1 12x1 4x1; do
  DFX_BWD_CFG=$c timeout 300 python bench.py $B > gpurun_out/bwdcfg_bench.log 2>&1
  echo "$c | $(tail -1 gpurun_out/bwdcfg_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels"]["compose_bwd_dmag"]["avg_us"])')" >> $O
done
done
cat $O
