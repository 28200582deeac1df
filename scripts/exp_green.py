"""Experiment: SM-partitioned pipelining with green contexts (norm on one SM partition,
compose kernels on the other), eager launches.  Analysis tool."""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(f"driver error {err}")
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


def main():
    import torch
    from cuda.bindings import driver as drv
    import paper_2603_22276_b200 as P
    norm_sms = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    budget = int(sys.argv[2]) if len(sys.argv) > 2 else norm_sms
    only = sys.argv[3] if len(sys.argv) > 3 else "both"     # both | norm | compose
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    chk(drv.cuInit(0))
    dev = chk(drv.cuDeviceGet(0))
    res = chk(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    print("total SMs", res.sm.smCount)
    groups, n, rem = drv.cuDevSmResourceSplitByCount(1, res, 0, norm_sms)[1:]
    print("split", groups[0].sm.smCount, rem.sm.smCount)
    def mk(r):
        desc = chk(drv.cuDevResourceGenerateDesc([r], 1))
        g = chk(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        st = chk(drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
        return g, st
    gA, sA = mk(groups[0])
    gB, sB = mk(rem)
    tsA = torch.cuda.ExternalStream(int(sA))
    tsB = torch.cuda.ExternalStream(int(sB))

    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    d_out = d_in = 8192
    r, rows = 384, 4096
    s = 2.0 / math.sqrt(r)
    cs, _ = P.plan_chunks(d_out, d_in)
    bf = torch.bfloat16
    nb = 4
    sets = []
    for i in range(nb):
        b = dict(W=torch.randn(d_out, d_in, device="cuda").to(bf), A=torch.randn(r, d_in, device="cuda").to(bf),
                 B=torch.randn(d_out, r, device="cuda").to(bf), base=torch.randn(rows, d_out, device="cuda").to(bf),
                 lora=torch.randn(rows, d_out, device="cuda").to(bf), dy=torch.randn(rows, d_out, device="cuda").to(bf))
        b.update(wn=torch.empty(d_out, device="cuda"), g=torch.empty(d_out, device="cuda"),
                 m=torch.ones(d_out, device="cuda") * 90, dm=torch.empty(d_out, device="cuda"))
        for k in ("delta", "inner", "dl", "db"):
            b[k] = torch.empty_like(b["base"])
        sets.append(b)
    torch.cuda.synchronize()

    def run(n):
        evn = [torch.cuda.Event() for _ in range(n)]
        evc = [torch.cuda.Event() for _ in range(n)]
        for i in range(n):
            b = sets[i % nb]
            with torch.cuda.stream(tsA):
                if i >= nb:
                    tsA.wait_event(evc[i - nb])
                if only in ("both", "norm"):
                    dfx.row_norm(b["W"], b["A"], b["B"], s, cs, b["wn"], m=b["m"], g=b["g"], stream=tsA)
                evn[i].record(tsA)
            with torch.cuda.stream(tsB):
                tsB.wait_event(evn[i])
                if only in ("both", "compose", "dual"):
                    dfx.compose_fwd(b["base"], b["lora"], b["g"], s, b["delta"], b["inner"], stream=tsB)
                if only in ("both", "compose", "bwd"):
                    dfx.compose_bwd(b["dy"], b["g"], s, b["dl"], b["db"], inner=b["inner"], w_norm=b["wn"],
                                    d_mag=b["dm"], stream=tsB)
                evc[i].record(tsB)
        return evc[n - 1]

    run(8)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    n = 200
    e0.record(tsA)
    last = run(n)
    tsA.wait_event(last)
    e1.record(tsA)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{only} norm_sms={norm_sms} budget={budget}: {ms / n * 1e3:.1f} us/module, {n / ms * 1e3:.0f} modules/s")


if __name__ == "__main__":
    main()
