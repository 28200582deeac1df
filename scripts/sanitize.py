"""Small-shape run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).
  compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    bf = torch.bfloat16
    for (d_out, d_in, r, rows, dt) in [(256, 512, 64, 100, bf), (384, 1024, 384, 64, bf),
                                      (136, 200, 24, 33, torch.float32), (520, 640, 40, 70, torch.float16)]:
        s = 2.0 / math.sqrt(r)
        cs, _ = P.plan_chunks(d_out, d_in)
        W, A, B = (torch.randn(*sh, device="cuda").to(dt) for sh in ((d_out, d_in), (r, d_in), (d_out, r)))
        wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        m = torch.ones(d_out, device="cuda")
        dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g)
        base, lora, dy = (torch.randn(rows, d_out, device="cuda").to(dt) for _ in range(3))
        delta, inner, dl, db = (torch.empty_like(base) for _ in range(4))
        dm = torch.empty(d_out, device="cuda")
        dfx.compose_fwd(base, lora, g, s, delta, inner)
        dfx.compose_bwd(dy, g, s, dl, db, inner=inner, w_norm=wn, d_mag=dm)
        if dt != torch.float32 and d_out % 8 == 0 and r % 8 == 0:
            mid = torch.randn(rows, r, device="cuda").to(dt)
            y = torch.empty_like(base)
            dfx.lora_compose(mid, B, base, g, s, y=y, inner=inner)
        for budget in (0, 24):
            dfx.set_sm_budget(budget)
            dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g)
        torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
