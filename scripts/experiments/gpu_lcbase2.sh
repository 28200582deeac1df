#!/bin/bash
# lora_compose, base staged by TMA (+ proxy fence): parity, then (slots, stages) per output count vs the register-prefetch kernel
O=gpurun_out/lcbase2.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_lora_compose.py -m gpu -q -x -p no:cacheprovider > gpurun_out/lcbase2_tests.log 2>&1; echo "tests rc=$?" >> $O; tail -2 gpurun_out/lcbase2_tests.log >> $O
DFX_LIB=variants/libdfx_lcold.so timeout 120 python scripts/lc_bench.py old >> $O 2>&1
for cfg in "0 0" "2 1" "3 1" "4 1" "2 2" "3 2" "1 2"; do
  set -- $cfg
  DFX_LC_SLOTS=$1 DFX_LC_STAGES=$2 timeout 120 python scripts/lc_bench.py "slots$1_stages$2" >> $O 2>&1
done
timeout 200 python scripts/lc_debug.py >> $O 2>&1
cat $O
