"""Per-kernel live times of the row norm (analysis tool, not the bench).
  python scripts/exp_norm_prof.py [--config c2] [--budget 0] [--iters 20]
Each call is queued behind a device spin so the CUDA-event brackets time the device."""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--r", type=int, default=0)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch
    import paper_2603_22276_b200 as P
    cfg = dict(bench.CONFIGS[a.config])
    if a.r:
        cfg["r"] = a.r
    d_out, d_in, r = cfg["d_out"], cfg["d_in"], cfg["r"]
    s = 2.0 / math.sqrt(r)
    dfx = P.Dfx(0)
    dfx.set_sm_budget(a.budget)
    cs, _ = P.plan_chunks(d_out, d_in)
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[cfg["dtype"]]
    sets = []
    for i in range(3):
        sets.append(dict(W=torch.randn(d_out, d_in, device="cuda").to(dt),
                         A=torch.randn(r, d_in, device="cuda").to(dt),
                         B=torch.randn(d_out, r, device="cuda").to(dt),
                         wn=torch.empty(d_out, device="cuda"), g=torch.empty(d_out, device="cuda"),
                         m=torch.ones(d_out, device="cuda") * 90.0))
    for d in sets:
        dfx.row_norm(d["W"], d["A"], d["B"], s, cs, d["wn"], m=d["m"], g=d["g"])
    torch.cuda.synchronize()
    dfx.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters)]
    for k in range(a.iters):
        torch.cuda._sleep(2_000_000)
        d = sets[k % 3]
        ev[k][0].record()
        dfx.row_norm(d["W"], d["A"], d["B"], s, cs, d["wn"], m=d["m"], g=d["g"])
        ev[k][1].record()
    rep = dfx.profile_report()
    dfx.profile(False)
    wall = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)[a.iters // 2]
    out = {"tag": a.tag, "config": a.config, "r": r, "budget": a.budget, "norm_wall_us": round(wall, 2),
           "commit_ummas": os.environ.get("DFX_COMMIT_UMMAS", "default")}
    for name, (n, tot, mn, mx) in rep.items():
        out[name] = round(tot / n * 1e3, 2)
    print(json.dumps(out), flush=True)
    dfx.close()


if __name__ == "__main__":
    main()
