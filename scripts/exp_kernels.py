"""Kernel-level timing for tuning experiments (analysis tool, not the bench).
  python scripts/exp_kernels.py [--config c2] [--what norm,bwd,fwd] [--iters 50]
Times each op alone on rotating buffer sets (> L2), CUDA events, median per call."""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--what", default="norm,bwd,fwd")
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch
    import paper_2603_22276_b200 as P
    cfg = bench.CONFIGS[a.config]
    d_out, d_in, r, rows = cfg["d_out"], cfg["d_in"], cfg["r"], cfg["tokens"]
    s = 2.0 / math.sqrt(r)
    dfx = P.Dfx(0)
    cs, _ = P.plan_chunks(d_out, d_in)
    bf = torch.bfloat16
    nb = 3
    sets = []
    for i in range(nb):
        d = dict(W=torch.randn(d_out, d_in, device="cuda").to(bf), A=torch.randn(r, d_in, device="cuda").to(bf),
                 B=torch.randn(d_out, r, device="cuda").to(bf), base=torch.randn(rows, d_out, device="cuda").to(bf),
                 lora=torch.randn(rows, d_out, device="cuda").to(bf),
                 mid=torch.randn(rows, r, device="cuda").to(bf))
        d.update(wn=torch.empty(d_out, device="cuda"), g=torch.ones(d_out, device="cuda") * 1.001,
                 m=torch.ones(d_out, device="cuda") * 90.0, delta=torch.empty_like(d["base"]),
                 inner=torch.empty_like(d["base"]), dl=torch.empty_like(d["base"]),
                 db=torch.empty_like(d["base"]), dm=torch.empty(d_out, device="cuda"))
        dfx.row_norm(d["W"], d["A"], d["B"], s, cs, d["wn"])
        sets.append(d)
    ops = {
        "norm": lambda d: dfx.row_norm(d["W"], d["A"], d["B"], s, cs, d["wn"], m=d["m"], g=d["g"]),
        "fwd": lambda d: dfx.compose_fwd(d["base"], d["lora"], d["g"], s, d["delta"]),
        "dual": lambda d: dfx.compose_fwd(d["base"], d["lora"], d["g"], s, d["delta"], d["inner"]),
        "bwd": lambda d: dfx.compose_bwd(d["base"], d["g"], s, d["dl"], d["db"], inner=d["lora"],
                                         w_norm=d["wn"], d_mag=d["dm"]),
    }
    ops["lora_fused"] = lambda d: dfx.lora_compose(d["mid"], d["B"], d["base"], d["g"], s,
                                                   y=d["dl"], inner=d["inner"])
    ops["lora_gemm_cublas"] = lambda d: torch.matmul(d["mid"], d["B"].T, out=d["lora"])
    out = []
    for w in a.what.split(","):
        f = ops[w]
        for i in range(6):
            f(sets[i % nb])
        torch.cuda.synchronize()
        ts = []
        batch = 12  # calls per event pair (hides host launch overhead)
        for i in range(a.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(1_000_000)
            e0.record()
            for j in range(batch):
                f(sets[(i + j) % nb])
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / batch)
        ts.sort()
        out.append(f"{w}={ts[len(ts) // 2]:.1f}us(min {ts[0]:.1f})")
    print(a.tag, a.config, " ".join(out), flush=True)


if __name__ == "__main__":
    main()
