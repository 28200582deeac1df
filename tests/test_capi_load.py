"""CPU checks of the drop-in boundary: the C ABI library loads and exports every entry
point include/dfx.h declares; host-only entry points work without a device; the
device entry points refuse to run without a B200 (no CPU fallback); the C++ drop-in
exports the reference API symbols."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2603_22276_b200 as P


def _declared(header):
    txt = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(dfx_\w+)\s*\(", txt, re.M)))


def test_header_declares_binding_surface():
    assert _declared(P.HEADER_PATH) == sorted(P.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    for name in _declared(P.HEADER_PATH):
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (dfx_\w+)", out))
    assert set(_declared(P.HEADER_PATH)) <= exported
    assert P.load_library().dfx_abi_version() == 1


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", P.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass  # tcgen05.mma in the norm kernel
    assert "UTMALDG" in sass                        # TMA tile loads
    assert "LDTM" in sass                           # tcgen05.ld epilogue


def test_plan_chunks_host_only():
    assert P.plan_chunks(8192, 8192) == (8192, 1)
    assert P.plan_chunks(28672, 8192) == (2304, 4)
    assert P.plan_chunks(4, 4) == (4, 1)
    with pytest.raises(P.DfxInvalidArgument):
        P.plan_chunks(1 << 20, 128, 1024)
    with pytest.raises(P.DfxInvalidArgument):
        P.plan_chunks(0, 8)


def test_no_device_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(P.DfxError) as e:
        P.Dfx(0)
    assert e.value.code in (P.DFX_ENODEV, P.DFX_ECUDA)


def test_dropin_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", P.DROPIN_PATH], capture_output=True,
                         text=True, check=True).stdout
    for sym in ["dorafactor::factored_norm_terms(", "dorafactor::assemble_norm(",
                "dorafactor::factored_row_norm(", "dorafactor::magnitude_scale(",
                "dorafactor::stable_compose(", "dorafactor::naive_compose(",
                "dorafactor::fused_compose(", "dorafactor::dual_output_compose(",
                "dorafactor::compose_backward(", "dorafactor::eager_traffic_model(",
                "dorafactor::plan_chunks(", "dorafactor::round_to_dtype(",
                "dorafactor::seeded_fixture(", "dorafactor::derive_seed("]:
        assert sym in out, sym


def test_dropin_throws_without_device():
    """The C++ drop-in's hot-path entry points fail loudly (std::runtime_error) without a GPU;
    host-only helpers (plan_chunks) still work.  Runs the conformance binary's filter."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    binary = os.path.join(P.ROOT_DIR, "tests", "cpp", "test_dropin")
    if not os.path.exists(binary):
        pytest.skip("conformance binary not built")
    r = subprocess.run([binary, "norm: rank-1"], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0
    assert "no usable sm_100 device" in r.stdout
