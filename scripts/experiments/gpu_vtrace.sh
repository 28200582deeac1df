#!/bin/bash
# V (G-stationary) per-CTA timeline, experiment build with -DDFX_TRACE.
mkdir -p gpurun_out/tr; rm -f gpurun_out/tr/v*.bin
for b in 0 138; do
  DFX_VTRACE=gpurun_out/tr/v_b$b.bin DFX_LIB=variants/libdfx_vtr.so timeout 120 python scripts/profile_module.py --steps 3 --budget $b > gpurun_out/tr/v_b$b.log 2>&1
  python scripts/trace_v.py gpurun_out/tr/v_b$b.bin > gpurun_out/tr/v_b$b.txt 2>&1
done
tail -3 gpurun_out/tr/v_b0.log
cat gpurun_out/tr/v_b*.txt
