#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_vkernel.py tests/test_gpu_norm_split.py tests/test_gpu_dsplit.py -q -x -p no:cacheprovider 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
mkdir -p gpurun_out/ko
run zs0 DFX_PAIR_ZSMEM=0
run zs1 DFX_PAIR_ZSMEM=1
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 40 --e2e-steps 0"
for rep in 1 2; do for v in 0 1; do
  DFX_PAIR_ZSMEM=$v timeout 300 python bench.py $B > /tmp/k.log 2>&1; echo "zsmem $v | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"], "U", d["kernels"]["u_rowdot_tc"]["avg_us"])')"
done; done
