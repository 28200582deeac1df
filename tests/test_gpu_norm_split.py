"""The split norm for pipelined stacks: dfx_norm_adapter (ba_sq from A and B alone) and
dfx_row_norm_ba (the W part finished with that ba_sq), against the oracle (pinned to the
reference), against the single dfx_row_norm call, and with an adapter call of one module
running concurrently with the W call of another on the same context (disjoint workspace)."""
import numpy as np
import pytest

from conftest import bits_equal, to_dev

pytestmark = pytest.mark.gpu


def _fixture(o, d_out, d_in, r, seed, dt):
    W = o.seeded_gaussian(d_out, d_in, o.derive_seed(seed, 0), dt)
    A = o.seeded_gaussian(r, d_in, o.derive_seed(seed, 1), dt)
    B = o.seeded_gaussian(d_out, r, o.derive_seed(seed, 2), dt)
    return W, A, B


@pytest.mark.parametrize("budget", [0, 140])
@pytest.mark.parametrize("d_out,d_in,r,dt", [(1024, 1024, 384, 1), (777, 640, 384, 1),
                                             (2048, 2048, 512, 1), (1000, 1024, 384, 2),
                                             (512, 4096, 64, 1)])
def test_split_matches_oracle_and_single_call(dfx, oracle, d_out, d_in, r, dt, budget):
    import torch
    o = oracle
    W, A, B = _fixture(o, d_out, d_in, r, 7 * d_out + r, dt)
    s = 2.0 / np.sqrt(r)
    cs, _ = o.plan_chunks(d_out, d_in)
    w, a, b = to_dev(W, dt), to_dev(A, dt), to_dev(B, dt)
    m = torch.from_numpy(np.abs(o.gaussian_vector(d_out, 1.0, 0.1, 5)).astype(np.float32)).cuda()
    dfx.set_sm_budget(budget)
    try:
        ba = torch.empty(d_out, device="cuda")
        dfx.norm_adapter(a, b, d_out, ba)
        wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        t = torch.empty(3, d_out, device="cuda")
        dfx.row_norm_ba(w, a, b, s, cs, ba, wn, m=m, g=g, terms=t)
        wn1, g1 = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        t1 = torch.empty(3, d_out, device="cuda")
        dfx.row_norm(w, a, b, s, cs, wn1, m=m, g=g1, terms=t1)
        torch.cuda.synchronize()
    finally:
        dfx.set_sm_budget(0)
    t, t1 = t.cpu().numpy(), t1.cpu().numpy()
    want = o.norm_terms(W, A, B, s, cs)
    assert bits_equal(t[0], want[0])                              # base_sq: the serial chain
    assert bits_equal(t[2], ba.cpu().numpy())                     # terms carry the given ba_sq
    scale_c = np.sqrt(want[0] * np.abs(want[2])) + 1e-30
    assert np.all(np.abs(t[1] - want[1]) <= 2e-5 * scale_c + 1e-6 * np.abs(want[1]))
    assert np.all(np.abs(t[2] - want[2]) <= 1e-4 * np.abs(want[2]) + 1e-6 * want[2].max())
    want_n = o.row_norm(dt, W, A, B, s, cs)
    ulp = np.spacing(want_n.astype(np.float32)) * (2 ** 16 if dt == 1 else 2 ** 13)
    assert np.all(np.abs(wn.cpu().numpy() - want_n) <= ulp)
    # the single call: the same W part bit for bit, ba_sq to the Gram's split-K order
    assert bits_equal(t[0], t1[0]) and bits_equal(t[1], t1[1])
    assert np.all(np.abs(t[2] - t1[2]) <= 1e-4 * np.abs(t1[2]) + 1e-6 * t1[2].max())
    want_g = o.magnitude_scale(dt, m.cpu().numpy(), wn.cpu().numpy())
    assert bits_equal(g.cpu().numpy(), want_g)


def test_adapter_overlaps_w_part(dfx, oracle):
    """Module j's adapter on one stream beside module i's W part on another (same context),
    repeatedly: every result equals the sequential one bit for bit."""
    import torch
    o = oracle
    d_out, d_in, r, dt = 2048, 2048, 384, 1
    s = 2.0 / np.sqrt(r)
    cs, _ = o.plan_chunks(d_out, d_in)
    mods = []
    for k in range(2):
        W, A, B = _fixture(o, d_out, d_in, r, 100 + k, dt)
        mods.append(dict(w=to_dev(W, dt), a=to_dev(A, dt), b=to_dev(B, dt),
                         ba=torch.empty(d_out, device="cuda"), wn=torch.empty(d_out, device="cuda")))
    for mm in mods:   # sequential reference
        dfx.norm_adapter(mm["a"], mm["b"], d_out, mm["ba"])
        dfx.row_norm_ba(mm["w"], mm["a"], mm["b"], s, cs, mm["ba"], mm["wn"])
    torch.cuda.synchronize()
    ref = [(mm["ba"].clone(), mm["wn"].clone()) for mm in mods]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for it in range(6):
        i, j = it % 2, (it + 1) % 2
        ba_j = torch.empty(d_out, device="cuda")
        wn_i = torch.empty(d_out, device="cuda")
        torch.cuda.synchronize()
        dfx.row_norm_ba(mods[i]["w"], mods[i]["a"], mods[i]["b"], s, cs, ref[i][0], wn_i,
                        stream=s1.cuda_stream)
        dfx.norm_adapter(mods[j]["a"], mods[j]["b"], d_out, ba_j, stream=s2.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(wn_i, ref[i][1]), it
        assert torch.equal(ba_j, ref[j][0]), it
