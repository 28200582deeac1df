#!/bin/bash
# G-stationary V kernel: norm tests forced on (DFX_V_GSTAT=1), per-kernel times, bench lines.
mkdir -p gpurun_out; O=gpurun_out/gstat.txt; : > $O
DFX_V_GSTAT=1 timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_dsplit.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gstat_tests.log 2>&1; echo "norm tests (gstat forced) rc=$?" >> $O; tail -3 gpurun_out/gstat_tests.log >> $O
for b in 0 104; do
  for v in "DFX_V_GSTAT=0" "DFX_V_GSTAT=1" "X=0"; do
    env $v DFX_PLAN_PRINT=1 timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$v" >> $O 2>&1
  done
done
for v in "DFX_V_GSTAT=0" "X=0"; do
  env $v timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/gstat_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/gstat_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "infer", d["variants"]["infer"]["value"], "U", d["roofline"]["avg_us"], d["roofline"]["unbudgeted"]["avg_us"], "norm", d["roofline_norm_stage"]["avg_us"], d["kernels"].get("ba_rowdot_tc"))')" >> $O
done
for ns in 84 92 104; do
  timeout 600 python bench.py --steps 400 --warmup 10 --norm-sms $ns --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/gstat_bench.log 2>&1
  echo "train norm-sms $ns | $(tail -1 gpurun_out/gstat_bench.log | cut -c1-150)" >> $O
done
cat $O
