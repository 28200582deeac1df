#!/bin/bash
bash scripts/gpu_round.sh r02k
SWEEP_OUT=gpurun_out/r02k_config_sweep.txt bash scripts/cfg_sweep.sh
for mode in train infer; do
  timeout 600 python bench.py --config c5 --mode $mode --steps 3 --warmup 3 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline > /tmp/c5.json 2>/tmp/c5.err
  echo "c5 $mode $(tail -1 /tmp/c5.json | cut -c1-200)" >> gpurun_out/r02k_config_sweep.txt
done
cat gpurun_out/r02k_config_sweep.txt
