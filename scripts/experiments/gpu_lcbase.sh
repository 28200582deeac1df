#!/bin/bash
# lora_compose with base staged by TMA (current) vs per-thread register prefetch (variants/libdfx_lcold.so)
O=gpurun_out/lcbase.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_lora_compose.py -m gpu -q -x -p no:cacheprovider > gpurun_out/lcbase_tests.log 2>&1; echo "tests rc=$?" >> $O; tail -2 gpurun_out/lcbase_tests.log >> $O
cat > /tmp/lcb.py <<'PY'
import sys, torch, math
sys.path.insert(0, '.')
import paper_2603_22276_b200 as P
dfx = P.Dfx(0)
rows, d_out, r = 4096, 8192, 384
mid = torch.randn(rows, r, device='cuda').bfloat16(); B = (0.05*torch.randn(d_out, r, device='cuda')).bfloat16()
base = torch.randn(rows, d_out, device='cuda').bfloat16(); g = torch.ones(d_out, device='cuda')
s = 2.0 / math.sqrt(r)
for outs in (("y", "inner"), ("y", "inner", "lora"), ("delta",), ("y",)):
    o = {k: torch.empty_like(base) for k in outs}
    f = lambda: dfx.lora_compose(mid, B, base, g, s, **o)
    for _ in range(5): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort(); us = ts[len(ts)//2]
    byts = (1 + len(outs)) * rows * d_out * 2 + (rows + d_out) * r * 2
    print(f"{sys.argv[1]} outs={'+'.join(outs)} {us:.1f} us {byts/us/1e3:.0f} GB/s")
PY
for lib in variants/libdfx_lcold.so paper_2603_22276_b200/libdfx.so; do
  DFX_LIB=$lib timeout 120 python /tmp/lcb.py $(basename $lib) >> $O 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lora_compose -s 3 -c 1 -o gpurun_out/lcbase_ncu python /tmp/lcb.py new > /dev/null 2>&1
cat $O
