#!/bin/bash
# V pair cap (DFX_V_PAIRS) in the pipelined C2 steps (training, inference), 400-step runs
mkdir -p gpurun_out; O=gpurun_out/vpairs.txt; : > $O
for rep in 1 2; do for vp in 0 16 24 32 48; do for mode in train infer; do
  DFX_V_PAIRS=$vp timeout 600 python bench.py --mode $mode --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/vp_bench.log 2>&1
  echo "vpairs $vp $mode | $(tail -1 gpurun_out/vp_bench.log | cut -c1-110)" >> $O
done; done; done
cat $O
