mkdir -p gpurun_out; rm -f gpurun_out/trace_*.bin
for b in 0 104; do
  DFX_LIB=variants/libdfx_trace.so DFX_TRACE=gpurun_out/trace_b$b.bin timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 3
done
for b in 0 104; do python scripts/trace_u.py gpurun_out/trace_b$b.bin; done
