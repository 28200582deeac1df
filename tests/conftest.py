import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

import pyoracle  # noqa: E402  (test infrastructure: the CPU checker)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session")
def oracle():
    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def reference():
    if not pyoracle.reference_available():
        pytest.skip("oracle/_ref (the compiled reference) not built here")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def dfx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_22276_b200 as P
    return P.Dfx(0)


def to_dev(a: np.ndarray, dtype_code: int):
    """float32 numpy (values representable in the dtype) -> torch CUDA tensor, exactly."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    return {0: t, 1: t.to(torch.bfloat16), 2: t.to(torch.float16)}[dtype_code]


def to_np(t) -> np.ndarray:
    return t.float().cpu().numpy()


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality of float32 arrays (NaN payloads compared as NaN)."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return np.array_equal(a.view(np.uint32)[~na], b.view(np.uint32)[~nb])
