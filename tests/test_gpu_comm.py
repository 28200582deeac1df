"""The symmetric-memory all-reduce (dfx_comm_* / dfx_norm_allreduce) on one
GPU.  `world` ranks live in this process, each with its own comm and its own stream; their
kernels run concurrently and meet at the device-flag barriers exactly as ranks on separate
GPUs do (peer pointers instead of IPC-mapped ones).  Checked: the result is the rank-order fp32
sum bitwise on every rank, repeated calls (epochs) and CUDA-graph replay stay correct, and the
d_in-split norm through partial -> dfx_norm_allreduce -> finish matches the single call."""
import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu


def _ranks(dfx, world, count):
    comms = [dfx.comm(k, world, count) for k in range(world)]
    bases = [c.base() for c in comms]
    for c in comms:
        c.set_peers(bases)
    return comms


def _rank_order_sum(parts):
    acc = parts[0].astype(np.float32).copy()
    for p in parts[1:]:
        acc = (acc + p.astype(np.float32)).astype(np.float32)
    return acc


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("count", [1, 7, 4096, 163840, 163843])
def test_allreduce_rank_order_bitwise(dfx, world, count):
    import torch
    comms = _ranks(dfx, world, count)
    streams = [torch.cuda.Stream() for _ in range(world)]
    rng = np.random.default_rng(count + world)
    outs = [torch.empty(count, device="cuda") for _ in range(world)]
    for rep in range(3):                       # several calls: per-block epochs advance
        parts = [rng.standard_normal(count).astype(np.float32) * (10.0 ** rng.integers(-3, 4))
                 for _ in range(world)]
        for c, p in zip(comms, parts):
            c.buffer().copy_(torch.from_numpy(p).cuda())
        torch.cuda.synchronize()
        for c, st, o in zip(comms, streams, outs):
            c.all_reduce(o, stream=st.cuda_stream)
        torch.cuda.synchronize()
        want = _rank_order_sum(parts)
        for o in outs:
            assert bits_equal(to_np(o), want)
    assert all(c.status() == 0 for c in comms)
    for c in comms:
        c.close()


def test_allreduce_in_cuda_graph(dfx):
    """Capturable: the epochs live in device memory, so graph replays keep the barriers in step."""
    import torch
    world, count = 2, 10000
    comms = _ranks(dfx, world, count)
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = [torch.empty(count, device="cuda") for _ in range(world)]
    src = [torch.randn(count, device="cuda") for _ in range(world)]
    graphs = []
    for c, st, o, x in zip(comms, streams, outs, src):
        c.all_reduce(o, stream=st.cuda_stream)           # eager once
    torch.cuda.synchronize()
    bufs = [c.buffer() for c in comms]                     # views made outside capture
    for c, st, o, x, b in zip(comms, streams, outs, src, bufs):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            b.copy_(x)
            c.all_reduce(o, stream=st.cuda_stream)
        graphs.append((g, st))
    torch.cuda.synchronize()
    for rep in range(5):
        for x in src:
            x.mul_(1.5)
        torch.cuda.synchronize()
        for g, st in graphs:
            with torch.cuda.stream(st):
                g.replay()
        torch.cuda.synchronize()
        want = _rank_order_sum([to_np(x) for x in src])
        for o in outs:
            assert bits_equal(to_np(o), want)
    assert all(c.status() == 0 for c in comms)
    for c in comms:
        c.close()


def test_allreduce_missing_peer_times_out(dfx):
    """A rank whose peer never arrives raises the error word after the bounded spin instead of
    hanging the GPU."""
    import torch
    comms = _ranks(dfx, 2, 64)
    out = torch.empty(64, device="cuda")
    comms[0].all_reduce(out)                  # rank 1 never calls
    torch.cuda.synchronize()
    assert comms[0].status() == 1
    for c in comms:
        c.close()


def test_allreduce_rejects_bad_arguments(dfx):
    import paper_2603_22276_b200 as P
    import torch
    with pytest.raises(P.DfxInvalidArgument):
        dfx.comm(2, 2, 16)
    with pytest.raises(P.DfxInvalidArgument):
        dfx.comm(0, 17, 16)
    c = dfx.comm(0, 2, 16)
    with pytest.raises(P.DfxInvalidArgument):     # peers not mapped yet
        c.all_reduce(torch.empty(16, device="cuda"))
    c.close()


@pytest.mark.parametrize("d_out,d_in,r,world,cs", [
    (2048, 8192, 384, 2, 4096),      # C2 d_in and rank, whole chunks per rank
    (1024, 8192, 384, 4, 2048),      # four ranks, one chunk each
    (768, 6912, 384, 3, 2304),       # C3's chunk size, three ranks
])
def test_dsplit_norm_through_symmetric_allreduce(dfx, oracle, d_out, d_in, r, world, cs):
    """The product path of the d_in split: dfx_norm_partial writes each rank's terms into its
    symmetric buffer, dfx_norm_allreduce sums them in rank order on every rank, dfx_norm_finish
    completes.  Every rank's norm is identical, within one bf16 ulp of the reference's, and
    base_sq is the reference's chunk loop bitwise when every rank after the first owns one
    chunk."""
    import torch
    from paper_2603_22276_b200 import dist as D
    W = oracle.seeded_gaussian(d_out, d_in, 41, 1)
    A = oracle.seeded_gaussian(r, d_in, 42, 1)
    B = oracle.seeded_gaussian(d_out, r, 43, 1)
    s = 2.0 / np.sqrt(r)
    Wd, Ad, Bd = to_dev(W, 1), to_dev(A, 1), to_dev(B, 1)
    n = r * r + 2 * d_out
    comms = _ranks(dfx, world, n)
    streams = [torch.cuda.Stream() for _ in range(world)]
    reds = [torch.empty(n, device="cuda") for _ in range(world)]
    wns = [torch.empty(d_out, device="cuda") for _ in range(world)]
    bounds = D.dsplit_bounds(d_in, world, cs)
    slices = [(Wd[:, k0:k1].contiguous(), Ad[:, k0:k1].contiguous()) for k0, k1 in bounds]
    torch.cuda.synchronize()
    for k in range(world):
        buf = comms[k].buffer()
        with torch.cuda.stream(streams[k]):
            dfx.norm_partial(slices[k][0], slices[k][1], Bd, cs, buf[: r * r],
                             buf[r * r: r * r + d_out], buf[r * r + d_out:])
    torch.cuda.synchronize()
    for k in range(world):
        comms[k].all_reduce(reds[k], stream=streams[k].cuda_stream)
    torch.cuda.synchronize()
    for k in range(world):
        red = reds[k]
        with torch.cuda.stream(streams[k]):
            dfx.norm_finish(Bd, red[: r * r], red[r * r: r * r + d_out], red[r * r + d_out:], s,
                            wns[k])
    torch.cuda.synchronize()
    assert all(c.status() == 0 for c in comms)
    for k in range(1, world):
        assert bits_equal(to_np(wns[k]), to_np(wns[0]))
    want = oracle.row_norm(1, W, A, B, s, cs)
    got = to_np(wns[0])
    assert np.all(np.abs(got - want) <= np.spacing(want.astype(np.float32)) * 2 ** 16)
    f64 = oracle.dense_row_norm_f64(W, A, B, s)
    assert np.max(np.abs(got - f64) / f64) <= 1e-2
    chunks_per_rank = [(k1 - k0 + cs - 1) // cs for k0, k1 in bounds]
    if all(c == 1 for c in chunks_per_rank[1:]):
        full_base = oracle.norm_terms(W, A, B, s, cs)[0]
        assert bits_equal(to_np(reds[0][r * r: r * r + d_out]), full_base)
    for c in comms:
        c.close()
