"""Fused LoRA-up + compose (dfx_lora_compose) at C2 per output set: median of 20 event-timed calls."""
import sys, torch, math
sys.path.insert(0, '.')
import paper_2603_22276_b200 as P
dfx = P.Dfx(0)
rows, d_out, r = 4096, 8192, 384
mid = torch.randn(rows, r, device='cuda').bfloat16(); B = (0.05*torch.randn(d_out, r, device='cuda')).bfloat16()
base = torch.randn(rows, d_out, device='cuda').bfloat16(); g = torch.ones(d_out, device='cuda')
s = 2.0 / math.sqrt(r)
OUTS = (("y", "inner"), ("y", "inner", "lora"), ("delta",), ("y",), ("y", "delta", "inner", "lora"))
for outs in OUTS:
    o = {k: torch.empty_like(base) for k in outs}
    f = lambda: dfx.lora_compose(mid, B, base, g, s, **o)
    try:
        f()
    except P.DfxError as e:
        print(f"{sys.argv[1]} outs={'+'.join(outs)} unsupported ({e})")
        continue
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
