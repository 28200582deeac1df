"""Runs the reference's hot-path unit tests restated against the C++ drop-in
(tests/cpp/test_dropin.cpp -> libdorafactor_b200.so -> libdfx.so) on the GPU."""
import os
import subprocess

import pytest

import paper_2603_22276_b200 as P

pytestmark = pytest.mark.gpu


def test_cpp_dropin_conformance():
    binary = os.path.join(P.ROOT_DIR, "tests", "cpp", "test_dropin")
    if not os.path.exists(binary):
        P.build()
    r = subprocess.run([binary], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed cases" in r.stdout
