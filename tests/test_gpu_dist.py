"""The d_in-split norm through the PRODUCT under a real world-size-2 process group: two
processes (both on cuda:0 — the box has one GPU), gloo rendezvous on 127.0.0.1, each rank
holding its K columns of W and A.  `dist.row_norm_dsplit` runs dfx_norm_partial ->
exchange -> dfx_norm_finish with the exchange done (a) by torch.distributed (gloo, staged
through host memory) and (b) by the library's symmetric-memory kernel over CUDA-IPC-mapped
peer buffers (`SymmetricAllReduce`).  Both ranks must produce identical norms and g, equal to
the single-call dfx_row_norm within one bf16 ulp, and (a) and (b) must agree bitwise (with two
ranks, a + b is the rank-order sum whichever way a library adds it)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, d_out, d_in, r, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_22276_b200 as P
    from paper_2603_22276_b200 import dist as D
    torch.cuda.set_device(0)
    dfx = P.Dfx(0)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234)                                  # the same module on both ranks
    bf = torch.bfloat16
    W = torch.randn(d_out, d_in, device="cuda", generator=gen).to(bf)
    A = (0.05 * torch.randn(r, d_in, device="cuda", generator=gen)).to(bf)
    B = (0.05 * torch.randn(d_out, r, device="cuda", generator=gen)).to(bf)
    m = torch.rand(d_out, device="cuda", generator=gen) + 0.5
    s = 2.0 / np.sqrt(r)
    cs, _ = P.plan_chunks(d_out, d_in, 2 ** 22)              # several chunks
    k0, k1 = D.dsplit_bounds(d_in, world, cs)[rank]
    Wk, Ak = W[:, k0:k1].contiguous(), A[:, k0:k1].contiguous()
    res = {}
    # (a) torch.distributed (gloo, host-staged)
    wn, g = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
    D.row_norm_dsplit(dfx, Wk, Ak, B, s, cs, wn, m=m, g=g)
    torch.cuda.synchronize()
    res["gloo"] = (wn.cpu().numpy(), g.cpu().numpy())
    # (b) the library's symmetric-memory all-reduce over IPC-mapped peer buffers
    comm = D.SymmetricAllReduce(dfx, r * r + 2 * d_out)
    for rep in range(3):
        wn2, g2 = torch.empty(d_out, device="cuda"), torch.empty(d_out, device="cuda")
        D.row_norm_dsplit(dfx, Wk, Ak, B, s, cs, wn2, m=m, g=g2, comm=comm)
        torch.cuda.synchronize()
    res["dfx"] = (wn2.cpu().numpy(), g2.cpu().numpy())
    res["status"] = comm.status()
    comm.close()
    # single call on the full matrices
    wn1 = torch.empty(d_out, device="cuda")
    dfx.row_norm(W, A, B, s, cs, wn1)
    torch.cuda.synchronize()
    res["single"] = wn1.cpu().numpy()
    res["launches"] = dfx.launches
    out_q.put((rank, res))
    tdist.barrier()
    tdist.destroy_process_group()
    dfx.close()


@pytest.mark.parametrize("d_out,d_in,r", [(1024, 8192, 384), (512, 4096, 64)])
def test_row_norm_dsplit_two_processes(d_out, d_in, r):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, d_out, d_in, r, q)) for k in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for k in (0, 1):
        assert got[k]["status"] == 0                      # no barrier timed out
        assert got[k]["launches"] > 0                     # the product's kernels ran
    for key in ("gloo", "dfx"):
        for i in (0, 1):
            assert np.array_equal(got[0][key][i].view(np.uint32), got[1][key][i].view(np.uint32))
    for i in (0, 1):
        assert np.array_equal(got[0]["gloo"][i].view(np.uint32), got[0]["dfx"][i].view(np.uint32))
    single = got[0]["single"]
    wn = got[0]["dfx"][0]
    assert np.all(np.abs(wn - single) <= np.spacing(single.astype(np.float32)) * 2 ** 16)
