"""GPU parity of the fused compose kernels (forward, dual output, backward) against the
CPU oracle (oracle/oracle.c, pinned to the reference by tests/test_oracle.py) and the
committed golden vectors produced by the reference itself (tests/golden/).

Bar: bitwise for delta / inner / d_lora / d_base / d_mag (the reference's arithmetic is
a fixed sequence of individually rounded fp32 ops; d_mag is a serial per-column chain,
SPEC.md:334), at ragged sizes and at BASELINE's full size (tokens=4096, d_out=8192)."""
import os

import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _g(o, n, dt, seed, sd=0.05):
    return np.array([o.round_to_dtype(v, dt) for v in o.gaussian_vector(n, 1.0, sd, seed)],
                    np.float32)


def _fwd(dfx, base, lora, g, s, dt, need_inner):
    import torch
    b, l = to_dev(base, dt), to_dev(lora, dt)
    gd = torch.from_numpy(g).cuda()
    d = torch.empty_like(b)
    i = torch.empty_like(b) if need_inner else None
    dfx.compose_fwd(b, l, gd, s, d, i)
    torch.cuda.synchronize()
    return to_np(d), (to_np(i) if need_inner else None)


@pytest.mark.parametrize("trial", range(60))
def test_path_parity_ragged(dfx, oracle, trial):
    """test_compose.cpp:94-114 — 60 ragged cases (d_out 1..200) in fp32/bf16/fp16."""
    o = oracle
    seed = o.derive_seed(12345, trial)
    rows = 1 + seed % 70
    d_out = 1 + o.derive_seed(seed, 1) % 200
    dt = trial % 3
    s = 0.0 if trial % 7 == 0 else 0.9
    base = o.gaussian_fixture(rows, d_out, 0.0, 3.0, o.derive_seed(seed, 2), dt)
    lora = o.gaussian_fixture(rows, d_out, 0.0, 3.0, o.derive_seed(seed, 3), dt)
    g = _g(o, d_out, dt, o.derive_seed(seed, 4))
    want_d, want_i = o.compose_fwd(dt, base, lora, g, s, need_inner=True)
    got_d, got_i = _fwd(dfx, base, lora, g, s, dt, need_inner=(trial % 2 == 0))
    assert bits_equal(got_d, want_d)
    if trial % 2 == 0:
        assert bits_equal(got_i, want_i)


def test_acceptance_criterion4_1000_cases(dfx, oracle):
    """acceptance.cpp:122-145 — 1,000 ragged cases (d_out 1..260), s in [-0.5, 1.5)."""
    o = oracle
    equal = 0
    for trial in range(1000):
        seed = o.derive_seed(77000, trial)
        rows = 1 + seed % 80
        d_out = 1 + o.derive_seed(seed, 1) % 260
        dt = trial % 3
        s = 0.0 if trial % 9 == 0 else -0.5 + 0.002 * (o.derive_seed(seed, 2) % 1000)
        base = o.gaussian_fixture(rows, d_out, 0.0, 4.0, o.derive_seed(seed, 3), dt)
        lora = o.gaussian_fixture(rows, d_out, 0.0, 4.0, o.derive_seed(seed, 4), dt)
        g = _g(o, d_out, dt, o.derive_seed(seed, 5))
        want, _ = o.compose_fwd(dt, base, lora, g, s)
        got_f, _ = _fwd(dfx, base, lora, g, s, dt, False)
        got_d, got_i = _fwd(dfx, base, lora, g, s, dt, trial % 2 == 0)
        equal += int(bits_equal(got_f, want) and bits_equal(got_d, want))
    assert equal == 1000


@pytest.mark.parametrize("dt", [0, 1, 2])
def test_full_size_forward_bitwise(dfx, oracle, dt):
    """BASELINE C2 compose shape (tokens=4096, d_out=8192), vectorised path, dual output."""
    rng = np.random.default_rng(20261017 + dt)
    rows, d_out = 4096, 8192
    base = rng.standard_normal((rows, d_out), dtype=np.float32)
    lora = rng.standard_normal((rows, d_out), dtype=np.float32)
    if dt:
        base, lora = to_np(to_dev(base, dt)), to_np(to_dev(lora, dt))
    g = _g(oracle, d_out, dt, 99, sd=0.0015)
    s = 2.0 / np.sqrt(384.0)
    want_d, want_i = oracle.compose_fwd(dt, base, lora, g, s, need_inner=True)
    got_d, got_i = _fwd(dfx, base, lora, g, s, dt, True)
    assert bits_equal(got_d, want_d)
    assert bits_equal(got_i, want_i)


def test_special_values_forward(dfx, oracle):
    """NaN / inf / subnormal / overflow propagate exactly as the reference's fp32 ops."""
    vals = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 1e-40, -3e-39, 3e38,
                     -3e38, 65504.0, 65520.0, 1e-8, 6e-8, 0.5], np.float32)
    for dt in (0, 1, 2):
        b = np.array([[oracle.round_to_dtype(v, dt) for v in vals]], np.float32)
        l = b[:, ::-1].copy()
        g = np.array([oracle.round_to_dtype(v, dt) for v in
                      [1.0, 0.5, 2.0, -1.0, 1.0, 1.0, 1.0, 1e-30, 1.0, 2.0, 0.0, 1.5, 1.0, 1.0,
                       3.0, np.inf]], np.float32)
        want_d, want_i = oracle.compose_fwd(dt, b, l, g, 0.9, need_inner=True)
        got_d, got_i = _fwd(dfx, b, l, g, 0.9, dt, True)
        assert bits_equal(got_d, want_d), dt
        assert bits_equal(got_i, want_i), dt


def _bwd(dfx, dy, g, s, inner, wn, dt, mag):
    import torch
    y = to_dev(dy, dt)
    gd = torch.from_numpy(g).cuda()
    dl, db = torch.empty_like(y), torch.empty_like(y)
    i = to_dev(inner, dt) if mag else None
    w = torch.from_numpy(wn).cuda() if mag else None
    dm = torch.empty(dy.shape[1], dtype=torch.float32, device="cuda") if mag else None
    dfx.compose_bwd(y, gd, s, dl, db, inner=i, w_norm=w, d_mag=dm)
    torch.cuda.synchronize()
    return to_np(dl), to_np(db), (dm.cpu().numpy() if mag else None)


@pytest.mark.parametrize("rows,d_out,dt", [(6, 10, 0), (1, 1, 1), (70, 37, 2), (1000, 512, 1),
                                           (333, 96, 0), (257, 264, 2), (4096, 8192, 1),
                                           (4096, 4096, 0), (0, 16, 1)])
def test_backward_bitwise(dfx, oracle, rows, d_out, dt):
    """compose.cpp:154-201 incl. the serial per-column d_mag chain, bitwise."""
    rng = np.random.default_rng(rows * 7 + d_out)
    dy = rng.standard_normal((rows, d_out), dtype=np.float32)
    inner = rng.standard_normal((rows, d_out), dtype=np.float32)
    if dt:
        dy, inner = to_np(to_dev(dy, dt)), to_np(to_dev(inner, dt))
    g = _g(oracle, d_out, dt, 7, sd=0.01)
    wn = np.array([oracle.round_to_dtype(5.0 + 0.01 * j, dt) for j in range(d_out)], np.float32)
    s = 0.7
    want = oracle.compose_bwd(dt, dy, g, s, inner, wn, mag_grad=True)
    got = _bwd(dfx, dy, g, s, inner, wn, dt, True)
    for w, gt in zip(want, got):
        assert bits_equal(gt, w)
    got_nomag = _bwd(dfx, dy, g, s, inner, wn, dt, False)
    assert bits_equal(got_nomag[0], want[0]) and bits_equal(got_nomag[1], want[1])


def test_backward_unit_g(dfx, oracle):
    """g == 1 zeroes d_base exactly (test_compose.cpp:167-177, acceptance.cpp:269-276)."""
    dy = oracle.gaussian_fixture(64, 256, 0.0, 1.0, 51, 1)
    g = np.ones(256, np.float32)
    dl, db, _ = _bwd(dfx, dy, g, 0.8, None, None, 1, False)
    assert not np.any(db)
    want = oracle.compose_bwd(1, dy, g, 0.8)
    assert bits_equal(db, want[1])  # signed zeros: (g-1)*dy keeps dy's sign
    assert bits_equal(dl, want[0])


def test_golden_compose(dfx):
    """Outputs of the reference itself (tests/golden/compose.npz, gen_golden.py)."""
    path = os.path.join(GOLDEN, "compose.npz")
    z = np.load(path)
    for k in range(int(z["n_cases"])):
        dt, s = int(z[f"c{k}_dt"]), float(z[f"c{k}_s"])
        base, lora, g = z[f"c{k}_base"], z[f"c{k}_lora"], z[f"c{k}_g"]
        got_d, got_i = _fwd(dfx, base, lora, g, s, dt, True)
        assert bits_equal(got_d, z[f"c{k}_delta"]), k
        assert bits_equal(got_i, z[f"c{k}_inner"]), k
    for k in range(int(z["n_bwd"])):
        dt, s = int(z[f"b{k}_dt"]), float(z[f"b{k}_s"])
        got = _bwd(dfx, z[f"b{k}_dy"], z[f"b{k}_g"], s, z[f"b{k}_inner"], z[f"b{k}_wn"], dt, True)
        assert bits_equal(got[0], z[f"b{k}_dlora"]), k
        assert bits_equal(got[1], z[f"b{k}_dbase"]), k
        assert bits_equal(got[2], z[f"b{k}_dmag"]), k


def test_invalid_arguments(dfx):
    import torch
    import paper_2603_22276_b200 as P
    y = torch.zeros(4, 8, device="cuda")
    g = torch.ones(8, device="cuda")
    with pytest.raises(P.DfxInvalidArgument):
        dfx.compose_bwd(y, g, 1.0, torch.empty_like(y), torch.empty_like(y), inner=None,
                        w_norm=g, d_mag=torch.empty(8, device="cuda"))
    with pytest.raises(P.DfxInvalidArgument):
        dfx.compose_fwd(y, y, None, 1.0, torch.empty_like(y))


@pytest.mark.parametrize("rows,d_out,dt", [(300, 264, 1), (4096, 1024, 1), (77, 40, 0), (129, 200, 2)])
def test_backward_magnitude_only(dfx, oracle, rows, d_out, dt):
    """dfx_compose_bwd with d_lora = d_base = NULL: the magnitude gradient alone, bitwise the
    reference's serial per-column chain (used after a row-chunked elementwise backward)."""
    import torch
    o = oracle
    seed = o.derive_seed(909, rows + d_out)
    dy = o.gaussian_fixture(rows, d_out, 0.0, 1.0, o.derive_seed(seed, 1), dt)
    inner = o.gaussian_fixture(rows, d_out, 0.0, 1.0, o.derive_seed(seed, 2), dt)
    g = _g(o, d_out, dt, o.derive_seed(seed, 3))
    wn = np.abs(_g(o, d_out, dt, o.derive_seed(seed, 4), sd=0.2)) + 0.5
    want = o.compose_bwd(dt, dy, g, 0.75, inner, wn, mag_grad=True)[2]
    dm = torch.empty(d_out, device="cuda")
    dfx.compose_bwd(to_dev(dy, dt), torch.from_numpy(g).cuda(), 0.75, None, None,
                    inner=to_dev(inner, dt), w_norm=torch.from_numpy(wn.astype(np.float32)).cuda(),
                    d_mag=dm)
    torch.cuda.synchronize()
    assert bits_equal(dm.cpu().numpy(), want)


def test_module_train_host_matches_device_path(dfx, oracle):
    """dfx_module_train_host (row-chunked H2D / compose / D2H, magnitude gradient last) returns
    exactly what the device-resident calls return."""
    import math
    import torch
    import paper_2603_22276_b200 as P
    d_out, d_in, r, rows = 512, 1024, 64, 2048
    s = 2.0 / math.sqrt(r)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    bf = torch.bfloat16
    rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=gen).to(bf)
    W, A, B, base, lora, dy = rnd(d_out, d_in), rnd(r, d_in), rnd(d_out, r), rnd(rows, d_out), \
        rnd(rows, d_out), rnd(rows, d_out)
    m = torch.rand(d_out, device="cuda", generator=gen) * 10 + 20
    cs, _ = P.plan_chunks(d_out, d_in)
    wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
    dfx.row_norm(W, A, B, s, cs, wn, m=m, g=g)
    delta, inner, dl, db = (torch.empty_like(base) for _ in range(4))
    dm = torch.empty(d_out, device="cuda")
    dfx.compose_fwd(base, lora, g, s, delta, inner)
    dfx.compose_bwd(dy, g, s, dl, db, inner=inner, w_norm=wn, d_mag=dm)
    torch.cuda.synchronize()
    h = {k: v.cpu().pin_memory() for k, v in dict(W=W, A=A, B=B, m=m, base=base, lora=lora, dy=dy).items()}
    out = {k: torch.empty_like(h["base"]).pin_memory() for k in ("delta", "dl", "db")}
    hdm = torch.empty(d_out).pin_memory()
    hg = torch.empty(d_out).pin_memory()
    dfx.module_train_host(P.BF16, h["W"], h["A"], h["B"], h["m"], h["base"], h["lora"], h["dy"], s,
                          d_out, d_in, r, rows, cs, out["delta"], out["dl"], out["db"], hdm, hg)
    assert torch.equal(hg, g.cpu())
    assert torch.equal(out["delta"], delta.cpu())
    assert torch.equal(out["dl"], dl.cpu())
    assert torch.equal(out["db"], db.cpu())
    assert torch.equal(hdm, dm.cpu())


@pytest.mark.parametrize("rows,d_out,dt", [(1000, 512, 1), (257, 264, 2), (4096, 8192, 1),
                                           (333, 96, 0), (64, 200, 1)])
def test_backward_bitwise_under_sm_budget(oracle, rows, d_out, dt):
    """With an SM budget set (composes beside the norm) the d_mag backward runs 256-byte
    column slabs; the results stay bitwise the reference's (compose.cpp:154-201)."""
    import paper_2603_22276_b200 as P
    dfx = P.Dfx(0)
    dfx.set_sm_budget(104)
    rng = np.random.default_rng(rows * 11 + d_out)
    dy = rng.standard_normal((rows, d_out), dtype=np.float32)
    inner = rng.standard_normal((rows, d_out), dtype=np.float32)
    if dt:
        dy, inner = to_np(to_dev(dy, dt)), to_np(to_dev(inner, dt))
    g = _g(oracle, d_out, dt, 9, sd=0.01)
    wn = np.array([oracle.round_to_dtype(5.0 + 0.01 * j, dt) for j in range(d_out)], np.float32)
    s = 0.7
    want = oracle.compose_bwd(dt, dy, g, s, inner, wn, mag_grad=True)
    got = _bwd(dfx, dy, g, s, inner, wn, dt, True)
    for w, gt in zip(want, got):
        assert bits_equal(gt, w)
    dfx.close()
