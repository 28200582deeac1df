#!/bin/bash
mkdir -p gpurun_out/tr; rm -f gpurun_out/tr/*.bin
for v in tr_skel tr_base; do for ka in 1 2; do
  DFX_PAIR_KA=$ka DFX_TRACE=gpurun_out/tr/${v}_ka$ka.bin DFX_LIB=variants/libdfx_$v.so timeout 120 python scripts/profile_module.py --steps 2 > /dev/null 2>&1
  python scripts/trace_u.py gpurun_out/tr/${v}_ka$ka.bin > gpurun_out/tr/${v}_ka$ka.txt 2>&1
done; done
DFX_PAIR_KA=2 DFX_TRACE=gpurun_out/tr/skel_d1024.bin DFX_LIB=variants/libdfx_tr_skel.so timeout 120 python scripts/profile_module.py --steps 2 --d-out 1024 > /dev/null 2>&1
python scripts/trace_u.py gpurun_out/tr/skel_d1024.bin > gpurun_out/tr/skel_d1024.txt 2>&1
head -50 gpurun_out/tr/*.txt
