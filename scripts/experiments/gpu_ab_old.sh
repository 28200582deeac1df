#!/bin/bash
# A/B: the pre-commit-group W.A^T kernel (44df44c) vs HEAD, norm alone and the bench step.
mkdir -p gpurun_out; O=gpurun_out/ab_old.txt; : > $O
for b in 0 104; do
  for v in old44 head cg1 cg2; do
    case $v in
      old44) E="DFX_LIB=variants/libdfx_old44.so";;
      head) E="X=0";;
      cg1) E="DFX_COMMIT_UMMAS=4";;
      cg2) E="DFX_COMMIT_UMMAS=8";;
    esac
    env $E timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag $v >> $O 2>&1
  done
done
for v in old44 head; do
  E=$([ $v = old44 ] && echo DFX_LIB=variants/libdfx_old44.so || echo X=0)
  env $E timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/ab_bench_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab_bench_$v.log | cut -c1-200)" >> $O
done
cat $O
