"""Multi-GPU plumbing for the DoRA hot path.

Three ways the path spreads over the GPUs of one box:

* **Module sharding** (the C5 layer stack): modules are independent, so each rank runs
  whole modules; `lpt_shards` balances them by cost (greedy longest-processing-time).
  No data-path collective.
* **Row split** of one module: a rank owns W / B / compose columns of a d_out block — the
  same kernels on a row slice, no exchange.
* **d_in split** (FSDP2 / TP-row style, the paper's stated gap): a rank
  owns W[:, K_k] and A[:, K_k].  The factored norm needs one exchange: the Gram G, base_sq
  and cross are sums over K, so each rank computes its slice's terms (`dfx_norm_partial`),
  ONE all-reduce sums {G [r*r], base_sq [d_out], cross [d_out]} (0.66 MB at r=384,
  d_out=8192), and every rank finishes locally (`dfx_norm_finish`: ba_sq = rowquad(B, G),
  assemble, round, magnitude).

The exchange runs either as the library's own symmetric-memory kernel
(`SymmetricAllReduce` over `dfx_norm_allreduce`: every rank reads every peer's partials over
NVLink and sums them in rank order, one launch, no host synchronisation) or through
torch.distributed (NCCL on GPUs; gloo, staged through host memory, in the tests).

K slices are aligned to the ChunkPlan so that each rank's base_sq chain covers whole chunks.
A rank's base_sq partial is the ascending-order sum of its chunks' serial partials, and the
exchange adds the ranks' partials in rank order, so the reduced base_sq is bitwise the
reference's `base_sq += partial` over chunks (factored_norm.cpp:52-60) exactly when every
rank after the first owns ONE chunk (e.g. two ranks, the second holding the last chunk);
otherwise fp32 addition is regrouped ((p0+p1)+(p2+p3) vs ((p0+p1)+p2)+p3) and base_sq agrees
to fp32 rounding (tests/test_gpu_dsplit.py checks both cases).
"""
from __future__ import annotations

import heapq
from typing import List, Sequence, Tuple


def module_cost(d_out: int, d_in: int, r: int, tokens: int, eb: int = 2) -> float:
    """Relative cost of one module on B200: tensor time of the norm + HBM time of the
    compose, in microseconds at the measured peaks (1388 TF/s sustained, 6554 GB/s)."""
    flops = 2.0 * d_out * d_in * r + 2.0 * r * r * d_in + 4.0 * d_out * r * r
    bytes_ = eb * (d_out * d_in + 3.0 * tokens * d_out)
    return flops / 1388e12 * 1e6 + bytes_ / 6554e9 * 1e6


def lpt_shards(costs: Sequence[float], n_ranks: int) -> List[List[int]]:
    """Greedy LPT: modules in decreasing cost, each to the least-loaded rank (ties: lowest
    rank, then lowest module index) — deterministic, within 4/3 of the optimum makespan."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, k) for k in range(n_ranks)]
    shards: List[List[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        load, k = heapq.heappop(heap)
        shards[k].append(i)
        heapq.heappush(heap, (load + costs[i], k))
    for sh in shards:
        sh.sort()
    return shards


def vlm32b_stack(hidden: int = 5120, mlp: int = 27648, layers: int = 64, kv_heads: int = 8,
                 head_dim: int = 128) -> List[Tuple[str, int, int]]:
    """The C5 inventory assumed by SURVEY sec. 8(d): 7 adapted modules per layer
    (q, k, v, o, gate, up, down) x 64 layers = 448 (d_out, d_in) modules."""
    kv = kv_heads * head_dim
    per_layer = [("q", hidden, hidden), ("k", kv, hidden), ("v", kv, hidden),
                 ("o", hidden, hidden), ("gate", mlp, hidden), ("up", mlp, hidden),
                 ("down", hidden, mlp)]
    return [(f"l{l}.{n}", o, i) for l in range(layers) for (n, o, i) in per_layer]


def row_split_bounds(d_out: int, world: int, align: int = 256) -> List[Tuple[int, int]]:
    """Row (d_out) ranges [r0, r1) per rank for the row split of one module: blocks of
    `align` rows (the 2-SM W.A^T kernel's pair tile), as even as the blocks allow.  Each rank
    runs the norm on W[r0:r1], B[r0:r1] with A replicated and the compose on columns
    [r0, r1) of the activations — no exchange (the Gram is recomputed per rank)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    units = (d_out + align - 1) // align
    out = []
    for k in range(world):
        u0, u1 = units * k // world, units * (k + 1) // world
        out.append((min(u0 * align, d_out), min(u1 * align, d_out)))
    return out


def dsplit_bounds(d_in: int, world: int, chunk_size: int) -> List[Tuple[int, int]]:
    """K ranges [k0, k1) per rank for the d_in split, on ChunkPlan chunk boundaries when
    there are at least `world` chunks (whole chunks per rank), else on 64-column
    boundaries (then base_sq is chunk-split and only tolerance-equal)."""
    n_chunks = (d_in + chunk_size - 1) // chunk_size
    unit = chunk_size if n_chunks >= world else 64
    units = (d_in + unit - 1) // unit
    out = []
    for k in range(world):
        u0, u1 = units * k // world, units * (k + 1) // world
        out.append((min(u0 * unit, d_in), min(u1 * unit, d_in)))
    return out


class SymmetricAllReduce:
    """The d_in split's exchange as one kernel over peer memory (include/dfx.h, dfx_comm_*).

    Each rank allocates a symmetric buffer of `count` fp32 through its Dfx context, the ranks
    swap CUDA IPC handles once through the process group (all_gather_object) and map each
    other's buffers; `buffer()` is where this rank writes its partial terms and
    `all_reduce(out)` writes the rank-order sum of all ranks' buffers into `out` (identical bits
    on every rank).  Without an initialised process group (one rank) it is a copy."""

    def __init__(self, dfx, count: int, group=None):
        import torch.distributed as tdist
        self.dist = tdist if (tdist.is_available() and tdist.is_initialized()) else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.count = count
        self.comm = dfx.comm(self.rank, self.world, count)
        if self.world > 1:
            handles = [None] * self.world
            self.dist.all_gather_object(handles, self.comm.ipc_handle(), group=group)
            self.comm.open(handles)
            self.dist.barrier(group=group)

    def buffer(self):
        return self.comm.buffer()

    def all_reduce(self, out, stream=None):
        self.comm.all_reduce(out, count=out.numel(), stream=stream)

    def status(self) -> int:
        return self.comm.status()

    def close(self):
        if self.comm is not None:
            if self.world > 1:
                self.dist.barrier(group=self.group)   # no peer still reads our buffer
            self.comm.close()
            self.comm = None


def row_norm_dsplit(dfx, W_k, A_k, B, s: float, chunk_size: int, w_norm, m=None, g=None,
                    terms=None, group=None, comm: "SymmetricAllReduce" = None):
    """d_in-split factored norm on this rank: partial terms -> one all-reduce -> finish.
    W_k / A_k are this rank's K columns (contiguous), B and m are replicated.  With `comm`
    the exchange is the library's symmetric-memory kernel; otherwise torch.distributed's
    all_reduce (staged through host memory when the group's backend is gloo).  Returns the
    reduced {G, base_sq, cross} buffer."""
    import torch
    import torch.distributed as tdist

    d_out, r = B.shape
    n = r * r + 2 * d_out
    buf = comm.buffer()[:n] if comm is not None else torch.empty(n, dtype=torch.float32,
                                                                  device=B.device)
    dfx.norm_partial(W_k, A_k, B, chunk_size, buf[: r * r], buf[r * r: r * r + d_out],
                     buf[r * r + d_out:])
    if comm is not None:
        red = torch.empty(n, dtype=torch.float32, device=B.device)
        comm.all_reduce(red)
    else:
        red = buf
        if tdist.is_available() and tdist.is_initialized():
            if tdist.get_backend(group) == "gloo":
                host = buf.cpu()
                tdist.all_reduce(host, op=tdist.ReduceOp.SUM, group=group)
                red.copy_(host)
            else:
                tdist.all_reduce(red, op=tdist.ReduceOp.SUM, group=group)
    dfx.norm_finish(B, red[: r * r], red[r * r: r * r + d_out], red[r * r + d_out:], s, w_norm,
                    m=m, g=g, terms=terms)
    return red
