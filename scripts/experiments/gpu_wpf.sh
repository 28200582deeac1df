#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/wpf.txt; : > $O
for w in 0 2 4 8 16 32; do
  DFX_W_PREFETCH=$w timeout 120 python scripts/exp_norm_prof.py --budget 0 --iters 20 --tag "wpf $w" >> $O 2>&1
done
for w in 0 8; do
  DFX_W_PREFETCH=$w timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/wpf_bench.log 2>&1
  echo "wpf $w | $(tail -1 gpurun_out/wpf_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"], "U", d["roofline"]["avg_us"])')" >> $O
done
cat $O
