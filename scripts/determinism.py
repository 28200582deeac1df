"""Run-to-run determinism of the row norm (bitwise): the same inputs N times, eager and in a
captured graph, under a given SM budget.  python scripts/determinism.py --budget 140 --reps 50"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--d-out", type=int, default=8192)
    ap.add_argument("--mix", default="", help="comma list of calls between the repeats: "
                    "cached, refresh, stream (plain norm on another stream), lora")
    a = ap.parse_args()
    import torch
    import paper_2603_22276_b200 as P
    d_out, d_in, r = a.d_out, 8192, 384
    s = 2.0 / math.sqrt(r)
    dfx = P.Dfx(0)
    dfx.set_sm_budget(a.budget)
    cs, _ = P.plan_chunks(d_out, d_in)
    torch.manual_seed(0)
    W = torch.randn(d_out, d_in, device="cuda").to(torch.bfloat16)
    A = torch.randn(r, d_in, device="cuda").to(torch.bfloat16)
    B = torch.randn(d_out, r, device="cuda").to(torch.bfloat16)
    m = torch.ones(d_out, device="cuda") * 90.0
    ref = None
    bad = 0
    cache = torch.empty(d_out, device="cuda")
    dfx.row_norm_cached(W, A, B, s, cs, cache, torch.empty(d_out, device="cuda"), refresh=True,
                        m=m, g=torch.empty(d_out, device="cuda"))
    other = torch.cuda.Stream()

    def mix():
        for kind in filter(None, a.mix.split(",")):
            wn2, g2 = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
            if kind == "cached":
                dfx.row_norm_cached(W, A, B, s, cs, cache, wn2, m=m, g=g2)
            elif kind == "refresh":
                dfx.row_norm_cached(W, A, B, s, cs, cache, wn2, refresh=True, m=m, g=g2)
            elif kind == "stream":
                with torch.cuda.stream(other):
                    dfx.row_norm(W, A, B, s, cs, wn2, m=m, g=g2)
            elif kind == "budget":
                dfx.set_sm_budget(0 if a.budget else 140)
                dfx.row_norm(W, A, B, s, cs, wn2, m=m, g=g2)
                dfx.set_sm_budget(a.budget)
        torch.cuda.synchronize()

    for i in range(a.reps):
        mix()
        wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        t = torch.empty(3, d_out, device="cuda")
        dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g, terms=t)
        torch.cuda.synchronize()
        cur = torch.cat([wn, g, t.flatten()]).view(torch.int32).clone()
        if ref is None:
            ref = cur
        elif not torch.equal(cur, ref):
            diff = (cur != ref).nonzero().flatten()
            bad += 1
            if bad <= 3:
                print(f"rep {i}: {diff.numel()} words differ, first {diff[:8].tolist()} "
                      f"(sections of {d_out}: wn, g, base, cross, ba)", flush=True)
    print(f"budget {a.budget} d_out {d_out} mix '{a.mix}': {bad} of {a.reps - 1} repeats differ "
          f"from the first", flush=True)


if __name__ == "__main__":
    main()
