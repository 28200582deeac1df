#!/bin/bash
# Knock-outs of the W.A^T pair kernel (ncu durations, isolated launches) + an L2-warm case.
mkdir -p gpurun_out/ko
for v in base ko_mma ko_chain ko_both ko_all; do
  L=$([ $v = base ] && echo paper_2603_22276_b200/libdfx.so || echo variants/libdfx_$v.so)
  DFX_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,gpc__cycles_elapsed.max --clock-control none -k regex:tc_pair_rowdot --csv \
     --log-file gpurun_out/ko/$v.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1
done
for cc in all none; do
  timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max --cache-control $cc --clock-control none -k regex:tc_pair_rowdot --csv \
     --log-file gpurun_out/ko/d4096_cache_$cc.csv python scripts/profile_module.py --d-out 4096 --steps 3 > /dev/null 2>&1
done
ls gpurun_out/ko
