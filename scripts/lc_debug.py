import sys, torch, math
sys.path.insert(0, '.')
import paper_2603_22276_b200 as P
dfx = P.Dfx(0)
rows, d_out, r = 4096, 8192, 384
gen = torch.Generator(device="cuda"); gen.manual_seed(11)
mid = torch.randn(rows, r, device="cuda", generator=gen).to(torch.bfloat16)
B = (0.05 * torch.randn(d_out, r, device="cuda", generator=gen)).to(torch.bfloat16)
base = torch.randn(rows, d_out, device="cuda", generator=gen).to(torch.bfloat16)
g = torch.ones(d_out, device="cuda")
s = 2.0 / math.sqrt(r)
for outs in (("inner", "lora"), ("y", "inner", "lora")):
    o = {k: torch.empty_like(base) for k in outs}
    dfx.lora_compose(mid, B, base, g, s, **o)
    torch.cuda.synchronize()
    want = (torch.tensor(s, dtype=torch.float32) * o["lora"].float() + base.float()).bfloat16()
    bad = (o["inner"] != want)
    n = int(bad.sum())
    print(outs, "mismatches", n)
    if n:
        idx = bad.nonzero()
        rr, cc = idx[:, 0], idx[:, 1]
        print(" rows tile (//128):", torch.unique(rr // 128)[:20].tolist(), " row%128 sample", torch.unique(rr % 128)[:20].tolist())
        print(" cols slice (//32):", torch.unique(cc // 32)[:20].tolist(), " tiles-n (//256):", torch.unique(cc // 256)[:10].tolist())
        print(" first", idx[:5].tolist())
