#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_lora_compose.py -q -x -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for v in lc1 head; do
  L=$([ $v = head ] && echo paper_2603_22276_b200/libdfx.so || echo variants/libdfx_$v.so)
  DFX_LIB=$L timeout 300 python scripts/exp_kernels.py --what lora_fused --iters 50 2>&1 | tail -1 | sed "s/^/$v: /"
done; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lora_compose --csv --log-file gpurun_out/lc_ncu.csv python scripts/exp_kernels.py --what lora_fused --iters 2 > /dev/null 2>&1
grep -v "^==" gpurun_out/lc_ncu.csv | tail -3
