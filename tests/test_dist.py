"""CPU tests of the multi-GPU host logic: LPT module sharding, chunk-aligned d_in split, and
dist.row_norm_dsplit's exchange over a real world_size-2 gloo process group (the two kernel
calls replaced by an oracle stand-in on this GPU-less box; the product runs the same helper
in tests/test_gpu_dist.py), checked against the oracle's full-matrix norm."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2603_22276_b200 import dist as D  # noqa: E402


def test_lpt_balance_and_coverage():
    stack = D.vlm32b_stack()
    assert len(stack) == 448
    costs = [D.module_cost(o, i, 384, 4096) for (_, o, i) in stack]
    for n in (1, 2, 4, 8):
        shards = D.lpt_shards(costs, n)
        flat = sorted(i for sh in shards for i in sh)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[i] for i in sh) for sh in shards]
        lower = max(sum(costs) / n, max(costs))
        assert max(loads) <= lower * 4 / 3 + 1e-9
        assert max(loads) / min(loads) < 1.01  # 448 modules balance almost perfectly
    assert D.lpt_shards([3, 3, 2, 2, 2], 2) == [[0, 2, 4], [1, 3]]


def test_dsplit_bounds():
    assert D.dsplit_bounds(8192, 2, 8192) == [(0, 4096), (4096, 8192)]       # 1 chunk: 64-col
    assert D.dsplit_bounds(8192, 4, 2304) == [(0, 2304), (2304, 4608), (4608, 6912), (6912, 8192)]
    b = D.dsplit_bounds(8192, 2, 2304)          # 4 chunks -> whole chunks per rank
    assert b == [(0, 4608), (4608, 8192)]
    for world in (1, 2, 3, 8):
        b = D.dsplit_bounds(1000, world, 1000)
        assert b[0][0] == 0 and b[-1][1] == 1000
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_row_split_bounds():
    assert D.row_split_bounds(8192, 2) == [(0, 4096), (4096, 8192)]
    assert D.row_split_bounds(8192, 8) == [(k * 1024, (k + 1) * 1024) for k in range(8)]
    b = D.row_split_bounds(28672, 3)
    assert b[0][0] == 0 and b[-1][1] == 28672 and all(x[0] % 256 == 0 for x in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(2))
    assert D.row_split_bounds(300, 4)[-1] == (256, 300)
    with pytest.raises(ValueError):
        D.row_split_bounds(10, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _OracleKernels:
    """CPU stand-in for the two Dfx calls row_norm_dsplit makes (norm_partial / norm_finish),
    computed with the oracle, so the helper's host logic — packed {G, base_sq, cross} layout,
    the gloo host-staged all-reduce, the finish from the reduced buffer — runs over a real
    world-2 process group on this GPU-less box.  The product itself runs the same helper in
    tests/test_gpu_dist.py (two processes on the GPU, gloo and the symmetric-memory kernel)."""

    def __init__(self, o):
        self.o = o

    def norm_partial(self, Wk, Ak, B, cs, gram, base, cross):
        Wk, Ak, B = (t.numpy() for t in (Wk, Ak, B))
        base_k, cross_k, _ = self.o.norm_terms(Wk, Ak, B, 1.0, cs)     # slice chain + cross
        gram.copy_(torch.from_numpy(
            (Ak.astype(np.float64) @ Ak.T.astype(np.float64)).astype(np.float32).ravel()))
        base.copy_(torch.from_numpy(base_k))
        cross.copy_(torch.from_numpy(cross_k))

    def norm_finish(self, B, gram, base, cross, s, w_norm, m=None, g=None, terms=None):
        r = B.shape[1]
        Bn = B.numpy().astype(np.float64)
        G = gram.numpy().reshape(r, r).astype(np.float64)
        ba = np.einsum("jl,lq,jq->j", Bn, G, Bn).astype(np.float32)
        w_norm.copy_(torch.from_numpy(self.o.assemble(np.ascontiguousarray(base.numpy()),
                                                      np.ascontiguousarray(cross.numpy()),
                                                      ba, 2 * s, s * s)))


def _dsplit_worker(rank, world, port, d_out, d_in, r, s, cs, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pyoracle
    o = pyoracle.Oracle()
    W = o.seeded_gaussian(d_out, d_in, 11)
    A = o.seeded_gaussian(r, d_in, 12)
    B = o.seeded_gaussian(d_out, r, 13)
    k0, k1 = D.dsplit_bounds(d_in, world, cs)[rank]
    Wk = torch.from_numpy(np.ascontiguousarray(W[:, k0:k1]))
    Ak = torch.from_numpy(np.ascontiguousarray(A[:, k0:k1]))
    wn = torch.empty(d_out)
    red = D.row_norm_dsplit(_OracleKernels(o), Wk, Ak, torch.from_numpy(B), s, cs, wn)
    norm = wn.numpy()
    base = red[r * r: r * r + d_out].numpy()
    if rank == 0:
        want = o.row_norm(0, W, A, B, s, cs)
        f64 = o.dense_row_norm_f64(W, A, B, s)
        full_base = o.norm_terms(W, A, B, s, cs)[0]
        out_q.put((float(np.max(np.abs(norm - want) / want)), float(np.max(np.abs(norm - f64) / f64)),
                   bool(np.array_equal(base, full_base))))
    dist.destroy_process_group()


@pytest.mark.parametrize("cs_mode", ["one_chunk", "two_chunks"])
def test_dsplit_exchange_gloo_world2(cs_mode):
    d_out, d_in, r, s = 96, 512, 16, 0.5
    cs = d_in if cs_mode == "one_chunk" else 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dsplit_worker, args=(k, 2, port, d_out, d_in, r, s, cs, q))
             for k in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    rel_ref, rel_f64, base_bitwise = q.get(timeout=10)
    assert rel_ref < 2e-5 and rel_f64 < 2e-5
    if cs_mode == "two_chunks":
        # whole chunks per rank: base_sq = (p0) + (p1) is the reference's chunk loop bitwise
        assert base_bitwise
