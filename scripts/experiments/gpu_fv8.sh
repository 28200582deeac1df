#!/bin/bash
# compose_fwd 256-bit variant (DFX_FWD_V8) vs the kept kernel: parity, standalone, pipelined steps
mkdir -p gpurun_out; O=gpurun_out/fv8.txt; : > $O
DFX_LIB=variants/libdfx_fv8.so timeout 600 python -m pytest tests/test_gpu_compose.py -q -x 2>&1 | tail -1 >> $O
for rep in 1 2; do for v in cur fv8; do
  echo "$v fwd: $(DFX_LIB=variants/libdfx_$v.so timeout 300 python scripts/exp_kernels.py --what fwd --iters 50 2>&1 | tail -2 | tr '\n' ' ')" >> $O
  for mode in train infer; do
    DFX_LIB=variants/libdfx_$v.so timeout 600 python bench.py --mode $mode --steps 400 --warmup 10 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 0 > gpurun_out/fv8_bench.log 2>&1
    echo "$v $mode | $(tail -1 gpurun_out/fv8_bench.log | cut -c60-100)" >> $O
  done
done; done
cat $O
