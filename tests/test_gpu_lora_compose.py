"""GPU parity of the fused LoRA-up GEMM + compose + residual kernel (dfx_lora_compose,
SURVEY 8(f) row 1) against the CPU oracle (oracle.c, pinned to the reference's
layer_forward by tests/test_oracle.py::test_layer_forward_pinned) and the reference's own
layer_forward (oracle/_ref).

Bar:
* given the kernel's own lora (returned as an output), delta / inner / y are BITWISE the
  reference's compose (compose.cpp:19-24, 131-137) and residual (layer.cpp:108-120);
* lora = round(mid . B^T) matches the reference's serial-k fp32 working_matmul within one
  working-dtype ulp plus the fp32 accumulation-order bound 2^-22 * k * sum|mid||B|
  (tensor-core summation order differs from the serial k loop);
* a whole layer forward (cuBLAS base / mid GEMMs, dfx_row_norm, dfx_lora_compose) agrees
  with the reference's layer_forward with cosine similarity > 0.9999 and a
  stated max-abs error."""
import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu


def _vec(o, n, dt, mean, sd, seed):
    return np.array([o.round_to_dtype(v, dt) for v in o.gaussian_vector(n, mean, sd, seed)],
                    np.float32)


def _run(dfx, mid, B, base, g, s, dt, bias=None, outs=("y", "inner", "lora")):
    import torch
    md, Bd, based = to_dev(mid, dt), to_dev(B, dt), to_dev(base, dt)
    gd = torch.from_numpy(g).cuda()
    bd = None if bias is None else torch.from_numpy(bias).cuda()
    o = {k: torch.empty_like(based) for k in outs}
    dfx.lora_compose(md, Bd, based, gd, s, bias=bd, **o)
    torch.cuda.synchronize()
    return {k: to_np(v) for k, v in o.items()}


def _lora_bound(o, mid, B, want, dt):
    ulp = np.spacing(np.abs(want).astype(np.float32)) * (2.0 ** 16 if dt == 1 else 2.0 ** 13)
    acc = np.abs(mid).astype(np.float64) @ np.abs(B).astype(np.float64).T
    return ulp + 2.0 ** -22 * mid.shape[1] * acc


CASES = [  # rows, d_out, r, dt
    (1, 8, 8, 1), (37, 136, 16, 1), (128, 256, 64, 1), (200, 264, 72, 1), (129, 520, 384, 1),
    (64, 1024, 128, 2), (255, 392, 40, 2), (300, 776, 384, 1),
    # several 256-row pair tiles, the last one's upper CTA entirely past the token tail
    (520, 1032, 384, 1), (777, 264, 64, 2),
    # d_out % 16 == 0 with a 16-column last tile (the 256-bit base loads' tail)
    (200, 272, 72, 1), (333, 1040, 384, 2),
]


@pytest.mark.parametrize("rows,d_out,r,dt", CASES)
def test_lora_compose_parity(dfx, oracle, rows, d_out, r, dt):
    o = oracle
    seed = o.derive_seed(4242, rows * 7 + d_out + r)
    mid = o.gaussian_fixture(rows, r, 0.0, 1.0, o.derive_seed(seed, 1), dt)
    B = o.gaussian_fixture(d_out, r, 0.0, 0.2, o.derive_seed(seed, 2), dt)
    base = o.gaussian_fixture(rows, d_out, 0.0, 2.0, o.derive_seed(seed, 3), dt)
    g = _vec(o, d_out, dt, 1.0, 0.05, o.derive_seed(seed, 4))
    bias = _vec(o, d_out, dt, 0.0, 0.5, o.derive_seed(seed, 5)) if rows % 2 else None
    s = 2.0 / np.sqrt(r)
    got = _run(dfx, mid, B, base, g, s, dt, bias)
    # compose + residual are bitwise given the kernel's lora
    want_d, want_i = o.compose_fwd(dt, base, got["lora"], g, s, need_inner=True)
    assert bits_equal(got["inner"], want_i)
    assert bits_equal(got["y"], o.residual(dt, base, want_d, bias))
    # delta output (a second call with another output set)
    got2 = _run(dfx, mid, B, base, g, s, dt, bias, outs=("delta", "lora"))
    assert bits_equal(got2["lora"], got["lora"]), "lora not deterministic across calls"
    assert bits_equal(got2["delta"], want_d)
    # the GEMM itself: within the working-dtype ulp + fp32 order bound of the reference's
    want_l = o.working_matmul_nt(dt, mid, B)
    assert np.all(np.abs(got["lora"] - want_l) <= _lora_bound(o, mid, B, want_l, dt))
    assert np.mean(got["lora"] == want_l) > 0.9


def test_lora_compose_full_size(dfx, oracle):
    """BASELINE C2 shape (tokens 4096, d_out 8192, r 384, bf16): bitwise compose +
    residual over all 33.5M elements given the kernel's lora; lora checked on 64 rows."""
    import torch
    o = oracle
    rows, d_out, r, dt = 4096, 8192, 384, 1
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    mid = torch.randn(rows, r, device="cuda", generator=gen).to(torch.bfloat16)
    B = (0.05 * torch.randn(d_out, r, device="cuda", generator=gen)).to(torch.bfloat16)
    base = torch.randn(rows, d_out, device="cuda", generator=gen).to(torch.bfloat16)
    g = (1.0 + 0.0015 * torch.randn(d_out, device="cuda", generator=gen)).to(torch.bfloat16).float()
    s = 2.0 / np.sqrt(r)
    y, inner, lora = (torch.empty_like(base) for _ in range(3))
    dfx.lora_compose(mid, B, base, g, s, y=y, inner=inner, lora=lora)
    torch.cuda.synchronize()
    base_h, lora_h, g_h = to_np(base), to_np(lora), g.cpu().numpy()
    want_d, want_i = o.compose_fwd(dt, base_h, lora_h, g_h, s, need_inner=True)
    assert bits_equal(to_np(inner), want_i)
    assert bits_equal(to_np(y), o.residual(dt, base_h, want_d))
    mid_h, B_h = to_np(mid[:64]), to_np(B)
    want_l = o.working_matmul_nt(dt, mid_h, B_h)
    assert np.all(np.abs(lora_h[:64] - want_l) <= _lora_bound(o, mid_h, B_h, want_l, dt))


def test_layer_forward_vs_reference(dfx, oracle, reference):
    """Whole layer_forward (layer.cpp:51-127) on the GPU: base = X W^T and mid = X A^T by
    cuBLAS (plain library GEMMs, fp32 accumulate, rounded to bf16), w_norm / g by
    dfx_row_norm, then dfx_lora_compose (lora GEMM + compose + residual + bias)."""
    import torch
    o, R = oracle, reference
    rows, d_in, d_out, r, dt = 96, 256, 384, 32, 1
    seed = 777
    x = o.gaussian_fixture(rows, d_in, 0.0, 1.0, o.derive_seed(seed, 1), dt)
    W = o.gaussian_fixture(d_out, d_in, 0.0, 0.05, o.derive_seed(seed, 2), dt)
    A = o.gaussian_fixture(r, d_in, 0.0, 0.05, o.derive_seed(seed, 3), dt)
    B = o.gaussian_fixture(d_out, r, 0.0, 0.05, o.derive_seed(seed, 4), dt)
    m = np.abs(o.gaussian_vector(d_out, 1.2, 0.1, o.derive_seed(seed, 5)))
    bias = _vec(o, d_out, dt, 0.0, 0.1, o.derive_seed(seed, 6))
    s = 2.0 / np.sqrt(r)
    ref = R.layer_forward(dt, x, W, A, B, s, m, bias.astype(np.float64))

    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    xd, Wd, Ad, Bd = (to_dev(v, dt) for v in (x, W, A, B))
    base = xd @ Wd.T
    mid = xd @ Ad.T
    cs, _ = o.plan_chunks(d_out, d_in)
    md = torch.from_numpy(np.array([o.round_to_dtype(v, dt) for v in m], np.float32)).cuda()
    wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
    dfx.row_norm(Wd, Ad, Bd, s, cs, wn, m=md, g=g)
    y, inner = torch.empty_like(base), torch.empty_like(base)
    dfx.lora_compose(mid, Bd, base, g, s, y=y, inner=inner, bias=torch.from_numpy(bias).cuda())
    torch.cuda.synchronize()
    y_h, ref_y = to_np(y).astype(np.float64), ref["y"].astype(np.float64)
    cos = float(np.dot(y_h.ravel(), ref_y.ravel()) /
                (np.linalg.norm(y_h) * np.linalg.norm(ref_y)))
    max_abs = float(np.max(np.abs(y_h - ref_y)))
    print(f"layer_forward vs reference: cos {cos:.8f}, max|dy| {max_abs:.3e}")
    assert cos > 0.9999
    assert max_abs <= 4 * float(np.max(np.spacing(np.abs(ref["y"]).astype(np.float32)))) * 2 ** 16
    # the norm and g match the reference's (tolerance / one bf16 ulp)
    assert np.all(np.abs(to_np(wn) - ref["w_norm"]) <= np.spacing(ref["w_norm"].astype(np.float32)) * 2 ** 16)


def test_lora_compose_rejects(dfx):
    import torch
    import paper_2603_22276_b200 as P
    a = torch.zeros(4, 8, device="cuda", dtype=torch.float32)
    g = torch.ones(8, device="cuda")
    with pytest.raises(P.DfxError):
        dfx.lora_compose(a, a, a, g, 1.0, y=a)          # fp32: not a tcgen05 kind::f16 type
    b = torch.zeros(4, 8, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(P.DfxError):
        dfx.lora_compose(b, b, b, g, 1.0, y=b, delta=b, inner=b, lora=b)   # > 3 outputs
    B8 = torch.zeros(8, 8, device="cuda", dtype=torch.bfloat16)        # d_out = r = 8: valid
    dfx.lora_compose(b, B8, b, g, 1.0, y=torch.empty_like(b))
    flat = torch.zeros(4 * 8 + 1, device="cuda", dtype=torch.bfloat16)
    mis = flat[1:].view(4, 8)                                           # 2-byte offset
    with pytest.raises(P.DfxInvalidArgument):
        dfx.lora_compose(b, B8, mis, g, 1.0, y=torch.empty_like(b))
    g12 = torch.ones(12, device="cuda")
    with pytest.raises(P.DfxInvalidArgument):
        dfx.lora_compose(b, B8, b, g12[1:9], 1.0, y=torch.empty_like(b))  # misaligned g
