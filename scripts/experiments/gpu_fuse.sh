#!/bin/bash
# Fused norm epilogues (Gram reduction in the Gram GEMM, finisher in the last U / V tile):
# norm GPU tests, A/B against DFX_NORM_FUSE=0, and the bench step.
mkdir -p gpurun_out; O=gpurun_out/fuse.txt; : > $O
timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_dsplit.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fuse_tests.log 2>&1; echo "norm tests rc=$?" >> $O; tail -2 gpurun_out/fuse_tests.log >> $O
for b in 0 104; do
  for v in fused unfused; do
    E=$([ $v = unfused ] && echo DFX_NORM_FUSE=0 || echo X=0)
    env $E timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag $v >> $O 2>&1
  done
done
for v in fused unfused; do
  E=$([ $v = unfused ] && echo DFX_NORM_FUSE=0 || echo X=0)
  env $E timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/fuse_bench_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/fuse_bench_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["variants"]["infer"]["value"], d["roofline"]["avg_us"], d["roofline_norm_stage"]["avg_us"])')" >> $O
done
cat $O
