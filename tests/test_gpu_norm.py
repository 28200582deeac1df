"""GPU parity of the factored row norm + magnitude scale against the CPU oracle (pinned
to the reference by tests/test_oracle.py), the reference's own golden vectors, and the
fp64 dense ground truth.

Bars (BASELINE north_star): row norms within 1e-5 relative in fp32 and 1e-2 in bf16.
fp32 rows with heavy cancellation (kappa = (base+|2s cross|+s^2 ba)/norm^2 large) are
held to max(1e-5, 64*kappa*2^-24), the bound the reference itself needs.
Bitwise where the reference's arithmetic is order-fixed: base_sq (serial chain per
ChunkPlan chunk), assemble_norm, magnitude_scale."""
import os

import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _terms(dfx, W, A, B, s, cs, dt):
    import torch
    w, a, b = to_dev(W, dt), to_dev(A, dt), to_dev(B, dt)
    out = torch.empty(3, W.shape[0], dtype=torch.float32, device="cuda")
    dfx.norm_terms(w, a, b, s, cs, out[0], out[1], out[2])
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    return o[0], o[1], o[2]


def _row_norm(dfx, W, A, B, s, cs, dt, m=None):
    import torch
    w, a, b = to_dev(W, dt), to_dev(A, dt), to_dev(B, dt)
    wn = torch.empty(W.shape[0], dtype=torch.float32, device="cuda")
    g = torch.empty_like(wn) if m is not None else None
    md = torch.from_numpy(np.asarray(m, np.float32)).cuda() if m is not None else None
    terms = torch.empty(3, W.shape[0], dtype=torch.float32, device="cuda")
    dfx.row_norm(w, a, b, s, cs, wn, m=md, g=g, terms=terms)
    torch.cuda.synchronize()
    return wn.cpu().numpy(), (g.cpu().numpy() if g is not None else None), terms.cpu().numpy()


def _kappa(o, W, A, B, s):
    # fp64 terms via the dense route on small shapes
    BA = B.astype(np.float64) @ A.astype(np.float64)
    W64 = W.astype(np.float64)
    base = (W64 * W64).sum(1)
    cross = (W64 * BA).sum(1)
    ba = (BA * BA).sum(1)
    n2 = base + 2 * s * cross + s * s * ba
    return (base + np.abs(2 * s * cross) + s * s * ba) / np.maximum(n2, 1e-300)


def _fixture(o, d_out, d_in, r, seed, dt=0):
    W = o.seeded_gaussian(d_out, d_in, o.derive_seed(seed, 0), dt)
    A = o.seeded_gaussian(r, d_in, o.derive_seed(seed, 1), dt)
    B = o.seeded_gaussian(d_out, r, o.derive_seed(seed, 2), dt)
    return W, A, B


def test_known_answers(dfx, oracle):
    W = np.zeros((2, 2), np.float32)
    A = np.array([[3, 4]], np.float32)
    B = np.array([[1], [2]], np.float32)
    wn, _, _ = _row_norm(dfx, W, A, B, 1.0, 2, 0)
    assert np.allclose(wn, [5.0, 10.0], rtol=1e-6)
    W = np.eye(4, dtype=np.float32)
    A, B = oracle.seeded_gaussian(2, 4, 3), oracle.seeded_gaussian(4, 2, 4)
    wn, _, _ = _row_norm(dfx, W, A, B, 0.0, 4, 0)
    assert np.all(wn == 1.0)


@pytest.mark.parametrize("dt", [0, 2])
def test_acceptance_criterion1_grid(dfx, oracle, dt):
    """acceptance.cpp:54-89: 300 instances, d_out/d_in in {3,17,64,96,257}, r in
    {1,2,8,33}, s in {0, 1, 2/sqrt(r)}: GPU vs the oracle's own result and vs fp64."""
    o = oracle
    dims, ranks = [3, 17, 64, 96, 257], [1, 2, 8, 33]
    seed = 10000
    worst_ref = worst_f64 = 0.0
    n = 0
    for d_out in dims:
        for d_in in dims:
            for r in ranks:
                for sm in range(3):
                    s = 0.0 if sm == 0 else (1.0 if sm == 1 else 2.0 / np.sqrt(r))
                    seed += 1
                    W, A, B = _fixture(o, d_out, d_in, r, seed, dt)
                    cs, _ = o.plan_chunks(d_out, d_in)
                    got, _, _ = _row_norm(dfx, W, A, B, s, cs, dt)
                    want = o.row_norm(dt, W, A, B, s, cs)
                    f64 = o.dense_row_norm_f64(W, A, B, s)
                    kap = _kappa(o, W, A, B, s)
                    rel_ref = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
                    rel_64 = np.abs(got - f64) / np.maximum(np.abs(f64), 1e-30)
                    tol = 1e-5 if dt == 0 else 2e-3
                    bound = np.maximum(tol, 64 * kap * 2.0 ** -24)
                    assert np.all(rel_64 <= bound), (d_out, d_in, r, s, rel_64.max())
                    assert np.all(rel_ref <= 2 * bound), (d_out, d_in, r, s, rel_ref.max())
                    if s == 0.0:
                        assert bits_equal(got, want)  # serial chain + sqrt, bitwise
                    worst_ref = max(worst_ref, rel_ref.max())
                    worst_f64 = max(worst_f64, rel_64.max())
                    n += 1
    assert n == 300
    print(f"criterion 1 ({'fp32' if dt == 0 else 'fp16'}): {n} instances, max rel err vs "
          f"reference {worst_ref:.2e}, vs fp64 {worst_f64:.2e}")


@pytest.mark.parametrize("d_out,d_in,r,cs", [(24, 80, 1, 80), (24, 80, 768, 80), (64, 257, 4, 64),
                                             (300, 1000, 12, 128), (129, 4096, 8, 4096)])
def test_base_sq_bitwise_fp32(dfx, oracle, d_out, d_in, r, cs):
    """base_sq is the reference's serial chunked chain, bitwise (factored_norm.cpp:52-61)."""
    W, A, B = _fixture(oracle, d_out, d_in, r, d_out + d_in + r)
    want = oracle.norm_terms(W, A, B, 1.0, cs)
    got = _terms(dfx, W, A, B, 1.0, cs, 0)
    assert bits_equal(got[0], want[0])
    np.testing.assert_allclose(got[1], want[1], rtol=1e-4, atol=1e-3 * np.abs(want[1]).max())
    np.testing.assert_allclose(got[2], want[2], rtol=1e-4, atol=1e-4 * np.abs(want[2]).max())


@pytest.mark.parametrize("dt", [1, 2])
@pytest.mark.parametrize("d_out,d_in,r", [(256, 512, 64), (1024, 1024, 384), (300, 640, 40),
                                          (128, 4096, 512), (1000, 2048, 128), (8192, 256, 16),
                                          (512, 8192, 1024),
                                          # d_in % 64 != 0: 2-D operand loads (no K-atom view),
                                          # two atoms per stage; odd K-block count: one atom
                                          (384, 1000, 96), (256, 960, 64)])
def test_tensor_core_path(dfx, oracle, d_out, d_in, r, dt):
    """tcgen05/TMA path, bf16 (kind::f16 with bf16 operands) and fp16 (kind::f16 with fp16
    operands, DTypeKind::FP16E, dtype.hpp:12): base_sq bitwise; cross/ba_sq vs the oracle's fp32
    terms; the dtype-rounded norm within one ulp of the working dtype of the reference's and
    within the reference's bar of fp64 (1e-2 bf16, 2e-3 fp16)."""
    assert dfx.uses_tensor_cores(dt, d_out, d_in, r)
    W, A, B = _fixture(oracle, d_out, d_in, r, 31 * d_out + r, dt=dt)
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    want = oracle.norm_terms(W, A, B, s, cs)
    m = np.abs(oracle.gaussian_vector(d_out, 1.0, 0.1, 5))
    wn, g, t = _row_norm(dfx, W, A, B, s, cs, dt, m=m)
    assert bits_equal(t[0], want[0])
    scale_c = np.sqrt(want[0] * np.abs(want[2])) + 1e-30       # Cauchy-Schwarz size of cross
    assert np.all(np.abs(t[1] - want[1]) <= 2e-5 * scale_c + 1e-6 * np.abs(want[1]))
    assert np.all(np.abs(t[2] - want[2]) <= 1e-4 * np.abs(want[2]) + 1e-6 * want[2].max())
    want_n = oracle.row_norm(dt, W, A, B, s, cs)
    ulp = np.spacing(want_n.astype(np.float32)) * (2 ** 16 if dt == 1 else 2 ** 13)
    assert np.all(np.abs(wn - want_n) <= ulp)
    want_g = oracle.magnitude_scale(dt, m, wn)                 # g given OUR norm: bitwise
    assert bits_equal(g, want_g)
    if d_out * d_in * r <= 2 ** 28:
        f64 = oracle.dense_row_norm_f64(W, A, B, s)
        assert np.max(np.abs(wn - f64) / f64) <= (1e-2 if dt == 1 else 2e-3)


@pytest.mark.parametrize("a_scale", [1e-3, 1.0, 40.0])
def test_fp16_gram_range(dfx, oracle, a_scale):
    """fp16 operands: the Gram A.A^T exceeds fp16's range at large A (diag ~ d_in * 1600 here)
    and underflows it at small A; the V GEMM's operand is G scaled by a power of two chosen
    from its diagonal (gram_split), undone exactly in the epilogue.  ba_sq keeps the fp32 bar."""
    d_out, d_in, r = 512, 4096, 128
    W, A, B = _fixture(oracle, d_out, d_in, r, 77, dt=2)
    A = (A * np.float32(a_scale)).astype(np.float16).astype(np.float32)
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    want = oracle.norm_terms(W, A, B, s, cs)
    _, _, t = _row_norm(dfx, W, A, B, s, cs, 2)
    assert bits_equal(t[0], want[0])
    assert np.all(np.isfinite(t[2]))
    assert np.all(np.abs(t[2] - want[2]) <= 1e-4 * np.abs(want[2]) + 1e-6 * want[2].max())


def test_full_size_c2_sampled_rows(dfx, oracle):
    """BASELINE C2 (8192^2, r=384, bf16) at full size: every row's base_sq bitwise vs the
    serial chain, and 256 sampled rows' terms vs the oracle run on those rows."""
    import torch
    d_out = d_in = 8192
    r = 384
    rng = np.random.default_rng(20261017)
    W = to_np(to_dev(rng.standard_normal((d_out, d_in), dtype=np.float32), 1))
    A = to_np(to_dev(rng.standard_normal((r, d_in), dtype=np.float32), 1))
    B = to_np(to_dev(rng.standard_normal((d_out, r), dtype=np.float32), 1))
    s = 2.0 / np.sqrt(r)
    cs, nc = oracle.plan_chunks(d_out, d_in)
    assert nc == 1
    t = np.stack(_terms(dfx, W, A, B, s, cs, 1))
    base_want = oracle.norm_terms(W, A, B, 0.0, cs)[0]          # s = 0: chain only
    assert bits_equal(t[0], base_want)
    rows = np.sort(rng.choice(d_out, 256, replace=False))
    sub = oracle.norm_terms(np.ascontiguousarray(W[rows]), A, np.ascontiguousarray(B[rows]), s, cs)
    scale_c = np.sqrt(sub[0] * sub[2])
    assert np.all(np.abs(t[1][rows] - sub[1]) <= 2e-5 * scale_c)
    assert np.all(np.abs(t[2][rows] - sub[2]) <= 1e-4 * sub[2])
    torch.cuda.synchronize()


def test_assemble_and_magnitude_bitwise(dfx, oracle):
    """assemble_norm (factored_norm.cpp:122-136) and magnitude_scale (:219-240) bitwise,
    including clamp, NaN, -0, eps floor and bf16/fp16 rounding."""
    import torch
    rng = np.random.default_rng(3)
    n = 4099
    base = np.abs(rng.standard_normal(n).astype(np.float32)) * 100
    cross = rng.standard_normal(n).astype(np.float32) * 50
    ba = np.abs(rng.standard_normal(n).astype(np.float32)) * 30
    base[:6] = [0.0, -0.0, np.nan, 1.0, 0.0, np.inf]
    cross[:6] = [-1.0, 0.0, 0.0, 0.0, 0.0, -np.inf]
    for two_s, s2 in [(2.0, 1.0), (2 * 0.1020620726159658, 0.1020620726159658 ** 2), (0.0, 0.0)]:
        want = oracle.assemble(base, cross, ba, two_s, s2)
        dev = [torch.from_numpy(x).cuda() for x in (base, cross, ba)]
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        dfx.assemble(dev[0], dev[1], dev[2], two_s, s2, out)
        torch.cuda.synchronize()
        assert bits_equal(out.cpu().numpy(), want)
    for dt in (0, 1, 2):
        wn = np.array([oracle.round_to_dtype(v, dt) for v in
                       np.concatenate([[0.0, np.nan, 1e-13, 1e-7, 3.0], np.abs(rng.standard_normal(500))])],
                      np.float32)
        m = rng.standard_normal(wn.shape[0]) * 2
        want = oracle.magnitude_scale(dt, m, wn)
        md = torch.from_numpy(m.astype(np.float32)).cuda()
        g = torch.empty(wn.shape[0], dtype=torch.float32, device="cuda")
        dfx.magnitude_scale(dt, md, torch.from_numpy(wn).cuda(), g)
        torch.cuda.synchronize()
        assert bits_equal(g.cpu().numpy(), want)


def test_golden_norm(dfx):
    """Terms and norms produced by the reference itself (tests/golden/norm.npz)."""
    z = np.load(os.path.join(GOLDEN, "norm.npz"))
    for k in range(int(z["n_cases"])):
        dt, s, cs = int(z[f"n{k}_dt"]), float(z[f"n{k}_s"]), int(z[f"n{k}_cs"])
        W, A, B = z[f"n{k}_W"], z[f"n{k}_A"], z[f"n{k}_B"]
        t = _terms(dfx, W, A, B, s, cs, dt)
        assert bits_equal(t[0], z[f"n{k}_base"]), k
        wn, _, _ = _row_norm(dfx, W, A, B, s, cs, dt)
        want = z[f"n{k}_norm"]
        f64 = z[f"n{k}_f64"]
        kap = z[f"n{k}_kappa"]
        tol = 1e-5 if dt == 0 else 1e-2
        bound = np.maximum(tol, 64 * kap * 2.0 ** -24)
        assert np.all(np.abs(wn - f64) / np.maximum(f64, 1e-30) <= bound), k
        assert np.all(np.abs(wn - want) / np.maximum(want, 1e-30) <= 2 * bound), k


def test_invalid_arguments(dfx):
    import torch
    import paper_2603_22276_b200 as P
    w = torch.zeros(8, 16, device="cuda")
    a = torch.zeros(2, 16, device="cuda")
    b = torch.zeros(8, 2, device="cuda")
    o = torch.empty(8, device="cuda")
    with pytest.raises(P.DfxInvalidArgument):
        dfx.norm_terms(w, a[:0], b, 1.0, 16, o, o, o)       # rank 0
    with pytest.raises(P.DfxInvalidArgument):
        dfx.norm_terms(w, a, b, 1.0, 0, o, o, o)            # bad chunk plan


@pytest.mark.parametrize("budget", [64, 24, 8])
@pytest.mark.parametrize("d_out,d_in,r", [(1024, 1024, 384), (128, 4096, 512), (2048, 2048, 384),
                                          (768, 4608, 320)])
def test_sm_budget_plans(oracle, budget, d_out, d_in, r):
    """dfx_ctx_set_sm_budget re-plans the norm GEMMs (a budget below two N-split rounds picks
    the full-r 2-SM tiling, two UMMAs per K step, W ingested once); the result keeps the
    same bar: base_sq bitwise, cross / ba_sq within the fp32 bound, norm within a bf16 ulp."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    W, A, B = _fixture(oracle, d_out, d_in, r, 17 * d_out + r + budget, dt=1)
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    want = oracle.norm_terms(W, A, B, s, cs)
    m = np.abs(oracle.gaussian_vector(d_out, 1.0, 0.1, 5))
    wn, g, t = _row_norm(dfx, W, A, B, s, cs, 1, m=m)
    assert bits_equal(t[0], want[0])
    scale_c = np.sqrt(want[0] * np.abs(want[2])) + 1e-30
    assert np.all(np.abs(t[1] - want[1]) <= 2e-5 * scale_c + 1e-6 * np.abs(want[1]))
    assert np.all(np.abs(t[2] - want[2]) <= 1e-4 * np.abs(want[2]) + 1e-6 * want[2].max())
    want_n = oracle.row_norm(1, W, A, B, s, cs)
    assert np.all(np.abs(wn - want_n) <= np.spacing(want_n.astype(np.float32)) * 2 ** 16)
    dfx.close()


@pytest.mark.parametrize("budget", [72, 104, 138])
def test_sm_budget_full_size_c2(oracle, budget):
    """C2 at full size under the pipelined bench's budgets (138 = the training step's since
    round 2: the all-SM W.A^T plan with the Gram on 10 side SMs and V after U; 104 / 72: the
    full-r 2-SM tiling beside the Gram and V): base_sq bitwise on every row."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    d_out = d_in = 8192
    r = 384
    rng = np.random.default_rng(7)
    W = to_np(to_dev(rng.standard_normal((d_out, d_in), dtype=np.float32), 1))
    A = to_np(to_dev(rng.standard_normal((r, d_in), dtype=np.float32), 1))
    B = to_np(to_dev(rng.standard_normal((d_out, r), dtype=np.float32), 1))
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    t = np.stack(_terms(dfx, W, A, B, s, cs, 1))
    assert bits_equal(t[0], oracle.norm_terms(W, A, B, 0.0, cs)[0])
    rows = np.sort(rng.choice(d_out, 128, replace=False))
    sub = oracle.norm_terms(np.ascontiguousarray(W[rows]), A, np.ascontiguousarray(B[rows]), s, cs)
    assert np.all(np.abs(t[1][rows] - sub[1]) <= 2e-5 * np.sqrt(sub[0] * sub[2]))
    assert np.all(np.abs(t[2][rows] - sub[2]) <= 1e-4 * sub[2])
    dfx.close()


@pytest.mark.parametrize("d_out,d_in,r,cs", [(256, 512, 64, None), (1024, 1024, 384, None),
                                             (300, 640, 40, None), (136, 2048, 512, None),
                                             (512, 1024, 128, 256), (384, 4096, 96, 1536)])
def test_fp32_tensor_core_path(dfx, oracle, d_out, d_in, r, cs):
    """fp32 weights on tcgen05 (3xTF32, fp32-class accumulation): base_sq bitwise (serial
    chain, chunk partials), cross / ba_sq within the fp32 bounds of the oracle's terms, the
    norm within max(1e-5, 64 kappa 2^-24) of fp64 — the reference's own bar."""
    assert dfx.uses_tensor_cores(0, d_out, d_in, r)
    W, A, B = _fixture(oracle, d_out, d_in, r, 7 * d_out + r, dt=0)
    s = 2.0 / np.sqrt(r)
    if cs is None:
        cs, _ = oracle.plan_chunks(d_out, d_in)
    want = oracle.norm_terms(W, A, B, s, cs)
    m = np.abs(oracle.gaussian_vector(d_out, 1.0, 0.1, 5))
    wn, g, t = _row_norm(dfx, W, A, B, s, cs, 0, m=m)
    assert bits_equal(t[0], want[0])
    scale_c = np.sqrt(want[0] * np.abs(want[2])) + 1e-30
    assert np.all(np.abs(t[1] - want[1]) <= 2e-5 * scale_c + 1e-6 * np.abs(want[1]))
    assert np.all(np.abs(t[2] - want[2]) <= 1e-4 * np.abs(want[2]) + 1e-6 * want[2].max())
    f64 = oracle.dense_row_norm_f64(W, A, B, s)
    kappa = _kappa(oracle, W, A, B, s)
    assert np.all(np.abs(wn - f64) <= np.maximum(1e-5, 64 * kappa * 2.0 ** -24) * f64)
    assert bits_equal(g, oracle.magnitude_scale(0, m, wn))


def test_fp32_c1_full_size(dfx, oracle):
    """BASELINE C1 (4096^2, r = 384, fp32) at full size on the 3xTF32 path: base_sq bitwise
    on every row, sampled rows' norms vs fp64 within the reference's bar."""
    d_out = d_in = 4096
    r = 384
    rng = np.random.default_rng(4)
    W = rng.standard_normal((d_out, d_in), dtype=np.float32)
    A = rng.standard_normal((r, d_in), dtype=np.float32)
    B = rng.standard_normal((d_out, r), dtype=np.float32)
    s = 2.0 / np.sqrt(r)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    wn, _, t = _row_norm(dfx, W, A, B, s, cs, 0)
    assert bits_equal(t[0], oracle.norm_terms(W, A, B, 0.0, cs)[0])
    rows = np.sort(rng.choice(d_out, 64, replace=False))
    Ws, Bs = np.ascontiguousarray(W[rows]), np.ascontiguousarray(B[rows])
    f64 = oracle.dense_row_norm_f64(Ws, A, Bs, s)
    kappa = _kappa(oracle, Ws, A, Bs, s)
    assert np.all(np.abs(wn[rows] - f64) <= np.maximum(1e-5, 64 * kappa * 2.0 ** -24) * f64)


@pytest.mark.parametrize("budget", [0, 80])
@pytest.mark.parametrize("d_out,d_in,r,dt", [(1024, 1024, 384, 1), (2048, 4096, 64, 1),
                                             (768, 4608, 320, 1), (8192, 8192, 384, 1)])
def test_row_norm_cached(oracle, budget, d_out, d_in, r, dt):
    """the cached ||W||^2_row of a frozen W.  The refresh call is
    the full norm and fills the cache with base_sq (bitwise the serial chain); the cached call
    runs W.A^T without the chain and gives bitwise the full call's w_norm and g while W is
    unchanged — with a new A and B too (the trainable factors move every step).  A W edited
    after the refresh is the caller's responsibility: the cached call then differs."""
    import torch
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    tdt = torch.bfloat16 if dt == 1 else torch.float16
    gen = torch.Generator(device="cuda")
    gen.manual_seed(d_out + r + budget)
    W = torch.randn(d_out, d_in, device="cuda", generator=gen).to(tdt)
    cs, _ = oracle.plan_chunks(d_out, d_in)
    s = 2.0 / np.sqrt(r)
    m = torch.rand(d_out, device="cuda", generator=gen) * 50 + 10
    cache = torch.full((d_out,), float("nan"), device="cuda")
    for step in range(2):
        A = (0.05 * torch.randn(r, d_in, device="cuda", generator=gen)).to(tdt)
        B = (0.05 * torch.randn(d_out, r, device="cuda", generator=gen)).to(tdt)
        wn0, g0 = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        terms = torch.empty(3, d_out, device="cuda")
        dfx.row_norm(W, A, B, s, cs, wn0, m=m, g=g0, terms=terms)
        wn1, g1 = torch.empty_like(wn0), torch.empty_like(g0)
        if step == 0:
            dfx.row_norm_cached(W, A, B, s, cs, cache, wn1, refresh=True, m=m, g=g1)
            torch.cuda.synchronize()
            assert bits_equal(to_np(cache), to_np(terms[0]))
        else:
            dfx.row_norm_cached(W, A, B, s, cs, cache, wn1, m=m, g=g1)
        torch.cuda.synchronize()
        assert bits_equal(to_np(wn1), to_np(wn0)), f"step {step}"
        assert bits_equal(to_np(g1), to_np(g0)), f"step {step}"
    W[0].mul_(2)
    fresh = torch.empty(d_out, device="cuda")
    dfx.row_norm(W, A, B, s, cs, fresh)
    stale = torch.empty(d_out, device="cuda")
    dfx.row_norm_cached(W, A, B, s, cs, cache, stale)
    torch.cuda.synchronize()
    assert to_np(stale)[0] != to_np(fresh)[0]
    assert bits_equal(to_np(stale)[1:], to_np(fresh)[1:])
    dfx.close()


def test_row_norm_cached_rejects(dfx):
    import torch
    import paper_2603_22276_b200 as P
    W = torch.zeros(256, 512, device="cuda")
    A, B = torch.zeros(16, 512, device="cuda"), torch.zeros(256, 16, device="cuda")
    c, wn = torch.zeros(256, device="cuda"), torch.zeros(256, device="cuda")
    with pytest.raises(P.DfxError):      # fp32: not the bf16 / fp16 tensor-core path
        dfx.row_norm_cached(W, A, B, 0.5, 512, c, wn)
    Wb, Ab, Bb = W.bfloat16(), A.bfloat16(), B.bfloat16()
    with pytest.raises(P.DfxError):      # s == 0 has no cross term to compute
        dfx.row_norm_cached(Wb, Ab, Bb, 0.0, 512, c, wn)
    with pytest.raises(P.DfxInvalidArgument):
        dfx.row_norm_cached(Wb, Ab, Bb, 0.5, 512, None, wn)   # no cache buffer


def test_norm_plan_reports_budget():
    """dfx_norm_plan reports the planner's SM split; it follows dfx_ctx_set_sm_budget."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    u_all, _, _ = dfx.norm_plan(8192, 8192, 384, 8192)
    for budget in (96, 80, 64, 24):
        dfx.set_sm_budget(budget)
        u, side, strat = dfx.norm_plan(8192, 8192, 384, 8192)
        assert 0 < u <= budget and u + side <= budget and strat in (0, 1, 2)
        assert u <= u_all
    with pytest.raises(P.DfxError):
        dfx.norm_plan(8192, 8192, 384, 8192, dtype=P.F32)
    dfx.close()


def _full_size_check(dfx, oracle, d_out, d_in, r, seed, n_rows=256, cs=None):
    """Full-size bf16 tensor-core norm: base_sq bitwise on EVERY row against the serial chunked
    chain; cross / ba_sq on n_rows sampled rows within the Cauchy-Schwarz fp32 bounds; the
    norm on those rows within one bf16 ulp of the reference's (oracle.row_norm)."""
    rng = np.random.default_rng(seed)
    W = to_np(to_dev(rng.standard_normal((d_out, d_in), dtype=np.float32), 1))
    A = to_np(to_dev(rng.standard_normal((r, d_in), dtype=np.float32), 1))
    B = to_np(to_dev(rng.standard_normal((d_out, r), dtype=np.float32), 1))
    s = 2.0 / np.sqrt(r)
    if cs is None:
        cs, _ = oracle.plan_chunks(d_out, d_in)
    assert dfx.uses_tensor_cores(1, d_out, d_in, r)
    wn, _, t = _row_norm(dfx, W, A, B, s, cs, 1)
    assert bits_equal(t[0], oracle.norm_terms(W, A, B, 0.0, cs)[0])      # s = 0: chain only
    rows = np.sort(rng.choice(d_out, n_rows, replace=False))
    Ws, Bs = np.ascontiguousarray(W[rows]), np.ascontiguousarray(B[rows])
    sub = oracle.norm_terms(Ws, A, Bs, s, cs)
    assert np.all(np.abs(t[1][rows] - sub[1]) <= 2e-5 * np.sqrt(sub[0] * sub[2]) + 1e-6 * np.abs(sub[1]))
    assert np.all(np.abs(t[2][rows] - sub[2]) <= 1e-4 * sub[2])
    want_n = oracle.row_norm(1, Ws, A, Bs, s, cs)
    assert np.all(np.abs(wn[rows] - want_n) <= np.spacing(want_n.astype(np.float32)) * 2 ** 16)
    return cs


@pytest.mark.parametrize("budget", [0, 104, 120])
def test_full_size_c3_four_chunks(oracle, budget):
    """BASELINE C3 (d_out = 28672, d_in = 8192, r = 384, bf16) at full size with the reference's
    own plan (2304, 4): K splits only on chunk boundaries, the base_sq chain reset every 2304
    columns, and the planner's pair tiling for this shape (full-r nh = 2 pairs and N-split
    pairs, depending on the SM budget)."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    cs, nc = oracle.plan_chunks(28672, 8192)
    assert (cs, nc) == (2304, 4)
    assert _full_size_check(dfx, oracle, 28672, 8192, 384, 28672 + budget) == 2304
    dfx.close()


@pytest.mark.parametrize("r", [64, 128, 512])
def test_full_size_c4_ranks(dfx, oracle, r):
    """BASELINE C4 high-rank sweep at d_out = d_in = 8192 (r = 384 is C2, r = 1024 is covered by
    test_bf16_tensor_core_path on 512 rows and the full-size sampled check below)."""
    _full_size_check(dfx, oracle, 8192, 8192, r, 8192 + r)


def test_full_size_c4_r1024(dfx, oracle):
    _full_size_check(dfx, oracle, 8192, 8192, 1024, 1024, n_rows=128)


@pytest.mark.parametrize("budget", [0, 40])
@pytest.mark.parametrize("d_out,d_in,r,cs", [(300, 4096, 96, 1024),     # 4 chunks
                                             (520, 6912, 384, 2304),    # 3 chunks (C3's cs)
                                             (256, 8192, 128, 1280),    # 6 + ragged last chunk
                                             (1000, 4608, 384, 768)])   # 6 chunks, ragged rows
def test_bf16_multi_chunk(oracle, budget, d_out, d_in, r, cs):
    """bf16 tensor-core norm with >= 3 ChunkPlan chunks at small d_out (explicit chunk sizes):
    base_sq is the reference's chunked chain bitwise (factored_norm.cpp:49-101)."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(budget)
    _full_size_check(dfx, oracle, d_out, d_in, r, d_out + cs + budget, n_rows=min(d_out, 256), cs=cs)
    dfx.close()


def test_fused_finisher_state_across_calls(dfx, oracle):
    """The fused finisher's per-block arrival counters return to zero after every call: plain,
    cached-refresh and cached norms, two SM budgets and a shape with a phantom pair half
    (d_out = 1000: the last 256-row pair tile covers 1024 rows) interleaved on one stream leave
    a later plain norm bitwise equal to the first one."""
    import torch
    torch.manual_seed(3)
    outs = []
    for d_out in (2048, 1000):
        d_in, r = 1024, 384
        W = torch.randn(d_out, d_in, device="cuda").to(torch.bfloat16)
        A = torch.randn(r, d_in, device="cuda").to(torch.bfloat16)
        B = torch.randn(d_out, r, device="cuda").to(torch.bfloat16)
        m = torch.ones(d_out, device="cuda")
        s = 2.0 / np.sqrt(r)
        cs, _ = oracle.plan_chunks(d_out, d_in)
        cache = torch.empty(d_out, device="cuda")

        def plain():
            wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
            dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g)
            return torch.cat([wn, g]).view(torch.int32).clone()

        for budget in (0, 140):
            dfx.set_sm_budget(budget)
            first = plain()
            for _ in range(3):
                wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
                dfx.row_norm_cached(W, A, B, s, cs, cache, wn, refresh=True, m=m, g=g)
                dfx.row_norm_cached(W, A, B, s, cs, cache, wn, m=m, g=g)
                assert torch.equal(plain(), first)
            outs.append(first)
    dfx.set_sm_budget(0)
    torch.cuda.synchronize()
