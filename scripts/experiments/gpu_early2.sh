#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 $EXTRA > /dev/null 2>&1; }
run early2_base X=0
EXTRA="--budget 104" run early2_b104 X=0
timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_vkernel.py tests/test_gpu_dsplit.py -q -x -p no:cacheprovider > gpurun_out/ko/early2_tests.log 2>&1; tail -1 gpurun_out/ko/early2_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/ko/early2_bench.log 2>&1
echo "early2 | $(tail -1 gpurun_out/ko/early2_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"], "U", d["roofline"]["avg_us"])')"
