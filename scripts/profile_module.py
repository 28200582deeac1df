"""Runs a few DoRA module steps (row_norm + compose) eagerly for ncu captures.
  python scripts/profile_module.py [--config c2] [--steps 3] [--bwd]"""
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--budget", type=int, default=0, help="dfx_ctx_set_sm_budget for the norm")
    ap.add_argument("--d-out", type=int, default=0, help="override the config's d_out (analysis)")
    ap.add_argument("--raw-alloc", action="store_true",
                    help="W / A in plain cudaMalloc memory (not the torch caching allocator)")
    ap.add_argument("--fill", default="randn", choices=["randn", "zeros", "bits"],
                    help="W / A contents (analysis: does the data change the kernel's time?)")
    a = ap.parse_args()
    import torch
    import paper_2603_22276_b200 as P
    cfg = bench.CONFIGS[a.config]
    d_out, d_in, r, rows = cfg["d_out"], cfg["d_in"], cfg["r"], cfg["tokens"]
    if a.d_out:
        d_out = a.d_out
    s = 2.0 / math.sqrt(r)
    dfx = P.Dfx(0)
    dfx.set_sm_budget(a.budget)
    cs, _ = P.plan_chunks(d_out, d_in)
    bf = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[cfg["dtype"]]
    W = torch.randn(d_out, d_in, device="cuda").to(bf)
    A = torch.randn(r, d_in, device="cuda").to(bf)
    if a.raw_alloc:   # plain cudaMalloc'd buffers, copied from the torch tensors
        import ctypes
        rt = ctypes.CDLL("libcudart.so")
        keep = []
        def raw_like(t):
            ptr = ctypes.c_void_p()
            assert rt.cudaMalloc(ctypes.byref(ptr), ctypes.c_size_t(t.numel() * 2)) == 0
            keep.append(ptr)

            class Raw:
                __cuda_array_interface__ = {"shape": tuple(t.shape), "typestr": "<i2",
                                            "data": (ptr.value, False), "version": 3}
            return torch.as_tensor(Raw(), device="cuda").view(t.dtype)
        W2, A2 = raw_like(W), raw_like(A)
        W2.copy_(W); A2.copy_(A); W, A = W2, A2
        print("raw cudaMalloc operands", W.data_ptr() % 4096, flush=True)
    if a.fill == "zeros":
        W.zero_(); A.zero_()
    elif a.fill == "bits":       # random bit patterns of finite bf16 values
        for t in (W, A):
            v = torch.randint(0, 1 << 15, t.shape, device="cuda", dtype=torch.int32)
            v = (v & 0x3FFF) | ((v & 0x4000) << 1)      # exponent below the inf/nan range, random sign
            t.copy_(v.to(torch.int16).view(torch.bfloat16))
    B = torch.randn(d_out, r, device="cuda").to(bf)
    base = torch.randn(rows, d_out, device="cuda").to(bf)
    lora = torch.randn(rows, d_out, device="cuda").to(bf)
    wn = torch.empty(d_out, device="cuda")
    g = torch.empty(d_out, device="cuda")
    m = torch.ones(d_out, device="cuda") * 90.0
    delta, inner = torch.empty_like(base), torch.empty_like(base)
    dl, db = torch.empty_like(base), torch.empty_like(base)
    dm = torch.empty(d_out, device="cuda")
    for _ in range(a.steps):
        dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g)
        dfx.compose_fwd(base, lora, g, s, delta, inner if a.bwd else None)
        if a.bwd:
            dfx.compose_bwd(base, g, s, dl, db, inner=inner, w_norm=wn, d_mag=dm)
    torch.cuda.synchronize()
    print("ok", dfx.launches)


if __name__ == "__main__":
    main()
