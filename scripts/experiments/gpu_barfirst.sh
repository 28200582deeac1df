#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
for ka in 1 2; do
  run s_barfirst_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_s_barfirst.so
  run b_barfirst_ka$ka DFX_PAIR_KA=$ka DFX_LIB=variants/libdfx_b_barfirst.so
done
DFX_LIB=variants/libdfx_b_barfirst.so timeout 600 python -m pytest tests/test_gpu_norm.py -q -x -k "tensor_core_path or full_size_c2" -p no:cacheprovider > gpurun_out/ko/barfirst_tests.log 2>&1; tail -1 gpurun_out/ko/barfirst_tests.log
