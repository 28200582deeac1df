#!/bin/bash
# last_arrival with one acq_rel atomic (default) vs a fence in every thread (-DDFX_FENCE_ALL):
# V trace, parity, live times, bench.
mkdir -p gpurun_out/tr; O=gpurun_out/fence.txt; : > $O
DFX_VTRACE=gpurun_out/tr/v3_b0.bin DFX_LIB=variants/libdfx_vtr3.so timeout 120 python scripts/profile_module.py --steps 3 > /dev/null 2>&1
python scripts/trace_v.py gpurun_out/tr/v3_b0.bin | tail -11 >> $O
timeout 1200 python -m pytest tests/test_gpu_vkernel.py tests/test_gpu_norm.py tests/test_gpu_norm_split.py tests/test_gpu_bench.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fence_tests.log 2>&1; echo "tests rc=$?" >> $O; tail -2 gpurun_out/fence_tests.log >> $O
for b in 0 138; do for lib in variants/libdfx_fenceall.so paper_2603_22276_b200/libdfx.so variants/libdfx_fenceall.so paper_2603_22276_b200/libdfx.so; do
  DFX_LIB=$lib timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag "$lib" >> $O 2>&1
done; done
B="--steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400"
for lib in variants/libdfx_fenceall.so paper_2603_22276_b200/libdfx.so variants/libdfx_fenceall.so paper_2603_22276_b200/libdfx.so; do
  DFX_LIB=$lib timeout 600 python bench.py $B > gpurun_out/fe_bench.log 2>&1
  echo "$lib | $(tail -1 gpurun_out/fe_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], "infer", d["variants"]["infer"]["value"], "U", d["kernels"]["u_rowdot_tc"]["avg_us"], "V", d["kernels"]["ba_rowdot_tc"]["avg_us"], "norm", d["roofline_norm_stage"]["avg_us"])')" >> $O
done
cat $O
