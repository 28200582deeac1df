#!/bin/bash
# V on half its pairs under an SM budget (DFX_V_HALF=1, default) vs all planned pairs (0):
# pipelined steps of every budgeted (config, mode) plus C2 inference (unbudgeted: unchanged)
mkdir -p gpurun_out; O=gpurun_out/vhalf.txt; : > $O
for rep in 1 2; do for vh in 1 0; do
  for cm in "c2 train" "c2 infer" "c3 train" "c3 infer" "c5 train"; do
    set -- $cm
    DFX_V_HALF=$vh timeout 900 python bench.py --config $1 --mode $2 --steps 200 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/vh_bench.log 2>&1
    echo "vhalf $vh $1 $2 | $(tail -1 gpurun_out/vh_bench.log | cut -c60-100)" >> $O
  done
done; done
cat $O
