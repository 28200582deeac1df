#!/bin/bash
# W L2 prefetch depth (DFX_W_PREFETCH) after the 3-D prefetch fix; training + inference 400-step runs
mkdir -p gpurun_out; O=gpurun_out/uknobs2.txt; : > $O
DFX_W_PREFETCH=2 timeout 600 python -m pytest tests/test_gpu_norm.py -q -x -k "full or c2 or budget" 2>&1 | tail -1 >> $O
for rep in 1 2; do for kv in "X=0" "DFX_W_PREFETCH=1" "DFX_W_PREFETCH=2" "DFX_W_PREFETCH=4"; do for mode in train infer; do
  env $kv timeout 600 python bench.py --mode $mode --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/uk.log 2>&1
  echo "$kv $mode rc=$? | $(tail -1 gpurun_out/uk.log | cut -c60-100)" >> $O
done; done; done
cat $O
