#!/bin/bash
# Pair-kernel K atoms per stage (DFX_PAIR_KA) x fused finisher (DFX_NORM_FUSE): norm tests,
# per-kernel live times, the bench step, and an ncu capture of U at ka=2.
mkdir -p gpurun_out; O=gpurun_out/ka.txt; : > $O
timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_dsplit.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ka_tests.log 2>&1; echo "norm tests rc=$?" >> $O; tail -2 gpurun_out/ka_tests.log >> $O
for b in 0 104; do
  for v in "DFX_PAIR_KA=1 DFX_NORM_FUSE=0" "DFX_PAIR_KA=1" "DFX_PAIR_KA=2" "DFX_PAIR_KA=2 DFX_W_PREFETCH=0"; do
    env $v timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$v" >> $O 2>&1
  done
done
for v in "DFX_PAIR_KA=1 DFX_NORM_FUSE=0" "DFX_PAIR_KA=1" "DFX_PAIR_KA=2"; do
  env $v timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/ka_bench.log 2>&1
  echo "$v | $(tail -1 gpurun_out/ka_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "infer", d["variants"]["infer"]["value"], "U", d["roofline"]["avg_us"], d["roofline"]["unbudgeted"]["avg_us"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done
DFX_PAIR_KA=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
    -o gpurun_out/ka2_ncu_tc_pair_rowdot python scripts/profile_module.py --steps 3 > /dev/null 2>&1
cat $O
