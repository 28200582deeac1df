#!/bin/bash
# stream priorities in the pipelined graphs (bench.py --stream-priority), 400-step runs, two repeats
mkdir -p gpurun_out; O=gpurun_out/prio.txt; : > $O
for rep in 1 2; do for pr in none compose norm; do for mode in train infer; do
  timeout 600 python bench.py --mode $mode --stream-priority $pr --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/pr.log 2>&1
  echo "$pr $mode rc=$? | $(tail -1 gpurun_out/pr.log | cut -c60-100)" >> $O
done; done; done
cat $O
