#!/bin/bash
# lora_compose knock-outs (DFX_LC_KO_*: no base loads / no TMA stores / no UMMAs) + ncu full capture
mkdir -p gpurun_out
for rep in 1 2; do for v in head kobase kostore kobs komma ahead2; do
  L=$([ $v = head ] && echo paper_2603_22276_b200/libdfx.so || echo variants/libdfx_$v.so)
  DFX_LIB=$L timeout 300 python scripts/lc_bench.py $v 2>&1 | grep outs
done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lora_compose -s 2 -c 1 \
    -o gpurun_out/lcko_ncu_lora_compose python scripts/exp_kernels.py --what lora_fused --iters 1 > /dev/null 2>&1
echo ncu rc=$?
