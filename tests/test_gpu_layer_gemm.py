"""GPU parity of dfx_working_matmul — the layer drop-in's GEMMs — against
the oracle's restatement of the reference's working_matmul (matrix.cpp:53-78 + rounded_to,
layer.cpp:15-17; pinned by tests/test_oracle.py): BITWISE, every output a serial fp32 chain
over k ascending, for the three operand layouts the layer uses (X.W^T, d_lora^T.mid,
d_lora.B) and ragged shapes around the 64 x 64 x 16 tiling."""
import time

import numpy as np
import pytest

from conftest import bits_equal, to_dev, to_np

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (5, 7, 3), (64, 64, 16), (65, 63, 17), (130, 200, 96), (257, 129, 1000),
          (33, 384, 2048)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("dt", [0, 1, 2])
def test_working_matmul_bitwise(dfx, oracle, m, n, k, dt):
    import torch
    o = oracle
    seed = o.derive_seed(515, m * 1000003 + n * 1009 + k + dt)
    a = o.gaussian_fixture(m, k, 0.0, 1.0, o.derive_seed(seed, 1), dt)
    bt = o.gaussian_fixture(n, k, 0.0, 1.0, o.derive_seed(seed, 2), dt)
    want = o.working_matmul_nt(dt, a, bt)
    ad, btd = to_dev(a, dt), to_dev(bt, dt)
    c = torch.empty(m, n, device="cuda", dtype=ad.dtype)
    dfx.working_matmul(ad, btd, c)                                   # a . bt^T
    torch.cuda.synchronize()
    assert bits_equal(to_np(c), want)
    # the same product from transposed storage: (a^T)^T . (bt^T) — strided operands
    at_d, b_d = ad.T.contiguous(), btd.T.contiguous()
    c2 = torch.empty_like(c)
    dfx.working_matmul(at_d, b_d, c2, trans_a=True, trans_b=False)
    torch.cuda.synchronize()
    assert bits_equal(to_np(c2), want)


def test_working_matmul_rate(dfx):
    """Throughput at a layer-sized product (informational; the serial order is the contract)."""
    import torch
    m, n, k = 4096, 1024, 4096
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    dfx.working_matmul(a, b, c)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dfx.working_matmul(a, b, c)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"working_matmul {m}x{n}x{k}: {dt * 1e3:.2f} ms, {2 * m * n * k / dt / 1e12:.1f} TFLOP/s (fp32 CUDA cores, serial k)")
    assert dt > 0
