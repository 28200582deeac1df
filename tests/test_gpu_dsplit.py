"""d_in-split factored norm through the C ABI on one GPU: K slices computed separately
(dfx_norm_partial), their {G, base_sq, cross} summed in rank order (what the all-reduce
does), finished with dfx_norm_finish — compared with the single-call dfx_row_norm, the CPU
oracle on the full matrices, and (whole-chunk slices, 2 ranks) bitwise base_sq."""
import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d_out,d_in,r,world,cs,dt", [
    (512, 2048, 64, 2, 1024, 1),      # tensor-core path, whole chunks per rank
    (512, 2048, 384, 4, 2048, 1),     # tensor-core path, chunk split across ranks
    (2048, 8192, 384, 2, 4096, 1),    # C2 d_in and rank, 2 ranks, whole chunks
    (100, 300, 12, 2, 300, 0),        # SIMT fp32 path
])
def test_dsplit_matches_single_call(dfx, oracle, d_out, d_in, r, world, cs, dt):
    import torch
    from paper_2603_22276_b200 import dist as D
    W = oracle.seeded_gaussian(d_out, d_in, 21, dt)
    A = oracle.seeded_gaussian(r, d_in, 22, dt)
    B = oracle.seeded_gaussian(d_out, r, 23, dt)
    s = 2.0 / np.sqrt(r)
    m = np.abs(oracle.gaussian_vector(d_out, 1.0, 0.1, 24)).astype(np.float32)
    Wd, Ad, Bd = to_dev(W, dt), to_dev(A, dt), to_dev(B, dt)
    md = torch.from_numpy(m).cuda()
    tot = torch.zeros(r * r + 2 * d_out, device="cuda")
    for (k0, k1) in D.dsplit_bounds(d_in, world, cs):
        buf = torch.empty_like(tot)
        dfx.norm_partial(Wd[:, k0:k1].contiguous(), Ad[:, k0:k1].contiguous(), Bd, cs,
                         buf[: r * r], buf[r * r: r * r + d_out], buf[r * r + d_out:])
        tot += buf
    wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
    terms = torch.empty(3, d_out, device="cuda")
    dfx.norm_finish(Bd, tot[: r * r], tot[r * r: r * r + d_out], tot[r * r + d_out:], s, wn,
                    m=md, g=g, terms=terms)
    wn1, g1 = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
    dfx.row_norm(Wd, Ad, Bd, s, cs, wn1, m=md, g=g1)
    torch.cuda.synchronize()
    got, one = wn.cpu().numpy(), wn1.cpu().numpy()
    want = oracle.row_norm(dt, W, A, B, s, cs)
    f64 = oracle.dense_row_norm_f64(W, A, B, s)
    tol = 1e-2 if dt == 1 else 2e-5
    assert np.max(np.abs(got - f64) / f64) <= tol
    ulp = np.spacing(want.astype(np.float32)) * (2 ** 16 if dt == 1 else 8)
    assert np.all(np.abs(got - want) <= ulp)
    assert np.all(np.abs(got - one) <= ulp)
    # g from our norm is the reference's magnitude_scale bitwise
    assert bits_equal(g.cpu().numpy(), oracle.magnitude_scale(dt, m, got))
    if world == 2 and d_in % (2 * cs) == 0:
        full_base = oracle.norm_terms(W, A, B, s, cs)[0]
        assert bits_equal(tot[r * r: r * r + d_out].cpu().numpy(), full_base)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("d_out,d_in,r", [(2048, 2048, 384), (1280, 4096, 128)])
def test_row_split_matches_single_call(dfx, oracle, world, d_out, d_in, r):
    """SURVEY 8(e) row split of one module (no exchange): each rank's norm on W[r0:r1],
    B[r0:r1] with A replicated, and the compose on its d_out columns.  base_sq is bitwise
    the single call's (serial chain per row), the norm within the bf16 bar, and the compose
    columns bitwise (elementwise given the same g)."""
    import torch
    from paper_2603_22276_b200 import dist as D
    gen = torch.Generator(device="cuda")
    gen.manual_seed(d_out + world)
    bf = torch.bfloat16
    W = torch.randn(d_out, d_in, device="cuda", generator=gen).to(bf)
    A = (0.05 * torch.randn(r, d_in, device="cuda", generator=gen)).to(bf)
    B = (0.05 * torch.randn(d_out, r, device="cuda", generator=gen)).to(bf)
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    wn, terms = torch.empty(d_out, device="cuda"), torch.empty(3, d_out, device="cuda")
    dfx.row_norm(W, A, B, s, cs, wn, terms=terms)
    base = torch.randn(512, d_out, device="cuda", generator=gen).to(bf)
    lora = torch.randn(512, d_out, device="cuda", generator=gen).to(bf)
    g = (1.0 + 0.01 * torch.randn(d_out, device="cuda", generator=gen)).to(bf).float()
    delta = torch.empty_like(base)
    dfx.compose_fwd(base, lora, g, s, delta)
    for (r0, r1) in D.row_split_bounds(d_out, world):
        n = r1 - r0
        wk, tk = torch.empty(n, device="cuda"), torch.empty(3, n, device="cuda")
        dfx.row_norm(W[r0:r1].contiguous(), A, B[r0:r1].contiguous(), s, cs, wk, terms=tk)
        dk = torch.empty(512, n, device="cuda", dtype=bf)
        dfx.compose_fwd(base[:, r0:r1].contiguous(), lora[:, r0:r1].contiguous(),
                        g[r0:r1].contiguous(), s, dk)
        torch.cuda.synchronize()
        assert bits_equal(to_np(tk[0]), to_np(terms[0, r0:r1]))
        want = to_np(wn[r0:r1])
        assert np.all(np.abs(to_np(wk) - want) <= np.spacing(want.astype(np.float32)) * 2 ** 16)
        assert bits_equal(to_np(dk), to_np(delta[:, r0:r1]))
