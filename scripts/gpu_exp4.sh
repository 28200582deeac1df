mkdir -p gpurun_out; rm -f gpurun_out/trace_ko*.bin
for b in 0 104; do
  DFX_LIB=variants/libdfx_trace_kochain.so DFX_TRACE=gpurun_out/trace_ko_b$b.bin timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 3
done
for b in 0 104; do python scripts/trace_u.py gpurun_out/trace_ko_b$b.bin | tail -8; done
