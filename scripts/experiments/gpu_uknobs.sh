#!/bin/bash
# W.A^T knobs on the final build: L2 prefetch depth of W, ring stages; training + inference 400-step runs
mkdir -p gpurun_out; O=gpurun_out/uknobs.txt; : > $O
for rep in 1 2; do for kv in "X=0" "DFX_W_PREFETCH=1" "DFX_W_PREFETCH=2" "DFX_PAIR_STAGES=3"; do for mode in train infer; do
  env $kv timeout 600 python bench.py --mode $mode --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/uk.log 2>&1
  echo "$kv $mode | $(tail -1 gpurun_out/uk.log | cut -c60-100)" >> $O
done; done; done
cat $O
