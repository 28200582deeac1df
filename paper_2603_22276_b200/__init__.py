"""B200-native DoRA hot path (arXiv 2603.22276): factored row norm, magnitude scale,
fused compose forward/backward, as hand-written sm_100a kernels behind a C ABI.

The product is native code:
  * ``libdfx.so``             — CUDA kernels + the C ABI declared in include/dfx.h
  * ``libdorafactor_b200.so`` — the reference's C++ API (namespace dorafactor) on top

This module is the thin Python binding used by the tests, smoke() and bench.py: it
loads ``libdfx.so`` through ctypes and passes torch device pointers and the current
CUDA stream.  There is no Python or CPU implementation of the path here — when the
library is missing or no sm_100 device is present every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

__all__ = ["Dfx", "build", "LIB_PATH", "DROPIN_PATH", "F32", "BF16", "F16", "DfxError"]

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("DFX_LIB", os.path.join(PKG_DIR, "libdfx.so"))   # DFX_LIB: A/B builds
DROPIN_PATH = os.path.join(PKG_DIR, "libdorafactor_b200.so")
HEADER_PATH = os.path.join(ROOT_DIR, "include", "dfx.h")

F32, BF16, F16 = 0, 1, 2
DFX_OK, DFX_EINVAL, DFX_ECUDA, DFX_ENOMEM, DFX_ENODEV, DFX_EUNSUPPORTED = range(6)
_ERR_NAMES = {1: "EINVAL", 2: "ECUDA", 3: "ENOMEM", 4: "ENODEV", 5: "EUNSUPPORTED"}


class DfxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"dfx {_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class DfxInvalidArgument(DfxError, ValueError):
    """Raised where the reference throws std::invalid_argument."""


def build(verbose: bool = False) -> None:
    """Compile libdfx.so, libdorafactor_b200.so and the C++ conformance binary in-tree."""
    cmd = ["make", "-C", os.path.join(PKG_DIR, "csrc"), "-j8"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)


_vp, _fp = C.c_void_p, C.POINTER(C.c_float)
_i64, _f64, _int = C.c_int64, C.c_double, C.c_int

# name -> (restype, argtypes); mirrors include/dfx.h one-for-one
SIGNATURES = {
    "dfx_abi_version": (_int, []),
    "dfx_last_error": (C.c_char_p, []),
    "dfx_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "dfx_ctx_destroy": (None, [_vp]),
    "dfx_ctx_launches": (_i64, [_vp]),
    "dfx_profile_enable": (_int, [_vp, _int]),
    "dfx_profile_report": (_int, [_vp, C.c_char_p, C.c_size_t]),
    "dfx_plan_chunks": (_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]),
    "dfx_norm_terms": (_int, [_vp, _int, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _i64,
                              _vp, _vp, _vp, _vp]),
    "dfx_assemble_norm": (_int, [_vp, _vp, _vp, _vp, _f64, _f64, _i64, _int, _vp, _vp]),
    "dfx_magnitude_scale": (_int, [_vp, _int, _vp, _vp, _i64, _vp, _vp]),
    "dfx_row_norm": (_int, [_vp, _int, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _i64, _vp, _int,
                            _vp, _vp, _vp, _vp]),
    "dfx_norm_plan": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "dfx_row_norm_cached": (_int, [_vp, _int, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _i64, _vp,
                                   _int, _vp, _int, _vp, _vp, _vp]),
    "dfx_norm_partial": (_int, [_vp, _int, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                _vp]),
    "dfx_norm_finish": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _i64, _i64, _f64, _vp, _int, _vp, _vp,
                               _vp, _vp]),
    "dfx_compose_fwd": (_int, [_vp, _int, _vp, _vp, _vp, _f64, _i64, _i64, _vp, _vp, _vp]),
    "dfx_compose_bwd": (_int, [_vp, _int, _vp, _vp, _f64, _vp, _vp, _i64, _i64, _vp, _vp, _vp,
                               _vp]),
    "dfx_module_fwd_host": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _i64, _i64,
                                   _i64, _i64, _i64, _vp, _vp]),
    "dfx_ctx_set_sm_budget": (_int, [_vp, _int]),
    "dfx_working_matmul": (_int, [_vp, _int, _vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64,
                                  _vp, _vp]),
    "dfx_lora_compose": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _f64, _vp, _i64, _i64, _i64, _vp,
                                _vp, _vp, _vp, _vp]),
    "dfx_module_train_host": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _i64,
                                     _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "dfx_norm_uses_tensor_cores": (_int, [_int, _i64, _i64, _i64]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdfx.so (no device needed).  Raises if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: run paper_2603_22276_b200.build() (there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _dtype_code(t) -> int:
    import torch
    return {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}[t.dtype]


class Dfx:
    """One dfx_ctx on one device.  Methods take torch CUDA tensors (or raw pointers)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        ctx = _vp()
        rc = self.lib.dfx_ctx_create(device, C.byref(ctx))
        self._check(rc)
        self.ctx = ctx
        self.device = device

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dfx_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != DFX_OK:
            msg = self.lib.dfx_last_error().decode()
            if rc == DFX_EINVAL:
                raise DfxInvalidArgument(rc, msg)
            raise DfxError(rc, msg)

    @property
    def launches(self) -> int:
        return int(self.lib.dfx_ctx_launches(self.ctx))

    # ----------------------------------------------------------------- norm
    def norm_terms(self, W, A, B, s, chunk_size, base_sq, cross, ba_sq, stream=None):
        d_out, d_in = W.shape
        r = A.shape[0]
        self._check(self.lib.dfx_norm_terms(self.ctx, _dtype_code(W), _ptr(W), _ptr(A), _ptr(B),
                                            d_out, d_in, r, float(s), int(chunk_size),
                                            _ptr(base_sq), _ptr(cross), _ptr(ba_sq),
                                            _stream(stream)))

    def row_norm(self, W, A, B, s, chunk_size, w_norm, m=None, g=None, terms=None,
                 mag_dtype=None, stream=None):
        d_out, d_in = W.shape
        r = A.shape[0]
        dt = _dtype_code(W)
        self._check(self.lib.dfx_row_norm(self.ctx, dt, _ptr(W), _ptr(A), _ptr(B), d_out, d_in, r,
                                          float(s), int(chunk_size), _ptr(m),
                                          dt if mag_dtype is None else mag_dtype, _ptr(w_norm),
                                          _ptr(g), _ptr(terms), _stream(stream)))

    def norm_plan(self, d_out, d_in, r, chunk_size, dtype=BF16):
        """(u_sms, side_sms, strategy) of the tensor-core norm under the current SM budget."""
        u, sd, st = C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.dfx_norm_plan(self.ctx, dtype, d_out, d_in, r, int(chunk_size),
                                           C.byref(u), C.byref(sd), C.byref(st)))
        return u.value, sd.value, st.value

    def row_norm_cached(self, W, A, B, s, chunk_size, base_sq_cache, w_norm, refresh=False,
                        m=None, g=None, mag_dtype=None, stream=None):
        """Opt-in cached ||W||^2_row for a frozen W (dfx_row_norm_cached)."""
        d_out, d_in = W.shape
        r = A.shape[0]
        dt = _dtype_code(W)
        self._check(self.lib.dfx_row_norm_cached(
            self.ctx, dt, _ptr(W), _ptr(A), _ptr(B), d_out, d_in, r, float(s), int(chunk_size),
            _ptr(base_sq_cache), 1 if refresh else 0, _ptr(m),
            dt if mag_dtype is None else mag_dtype, _ptr(w_norm), _ptr(g), _stream(stream)))

    def norm_partial(self, W_k, A_k, B, chunk_size, gram, base_sq, cross, stream=None):
        """d_in-split step 1: this rank's K-slice terms (sum them over ranks)."""
        d_out, d_in_k = W_k.shape
        r = A_k.shape[0]
        self._check(self.lib.dfx_norm_partial(self.ctx, _dtype_code(W_k), _ptr(W_k), _ptr(A_k),
                                              _ptr(B), d_out, d_in_k, r, int(chunk_size),
                                              _ptr(gram), _ptr(base_sq), _ptr(cross),
                                              _stream(stream)))

    def norm_finish(self, B, gram, base_sq, cross, s, w_norm, m=None, g=None, terms=None,
                    mag_dtype=None, stream=None):
        """d_in-split step 2 from the reduced {gram, base_sq, cross}."""
        d_out, r = B.shape
        dt = _dtype_code(B)
        self._check(self.lib.dfx_norm_finish(self.ctx, dt, _ptr(B), _ptr(gram), _ptr(base_sq),
                                             _ptr(cross), d_out, r, float(s), _ptr(m),
                                             dt if mag_dtype is None else mag_dtype, _ptr(w_norm),
                                             _ptr(g), _ptr(terms), _stream(stream)))

    def assemble(self, base_sq, cross, ba_sq, two_s, s2, out, round_to=F32, n=None,
                 stream=None):
        n = base_sq.shape[0] if n is None else n
        self._check(self.lib.dfx_assemble_norm(self.ctx, _ptr(base_sq), _ptr(cross), _ptr(ba_sq),
                                               float(two_s), float(s2), n, round_to, _ptr(out),
                                               _stream(stream)))

    def magnitude_scale(self, dtype, m, w_norm, g, n=None, stream=None):
        n = m.shape[0] if n is None else n
        self._check(self.lib.dfx_magnitude_scale(self.ctx, dtype, _ptr(m), _ptr(w_norm), n,
                                                 _ptr(g), _stream(stream)))

    # -------------------------------------------------------------- compose
    def compose_fwd(self, base, lora, g, s, delta, inner=None, stream=None, dtype=None,
                    rows=None, d_out=None):
        rows = base.shape[0] if rows is None else rows
        d_out = base.shape[1] if d_out is None else d_out
        dt = _dtype_code(base) if dtype is None else dtype
        self._check(self.lib.dfx_compose_fwd(self.ctx, dt, _ptr(base), _ptr(lora), _ptr(g),
                                             float(s), rows, d_out, _ptr(delta), _ptr(inner),
                                             _stream(stream)))

    def compose_bwd(self, dy, g, s, d_lora, d_base, inner=None, w_norm=None, d_mag=None,
                    stream=None, dtype=None, rows=None, d_out=None):
        rows = dy.shape[0] if rows is None else rows
        d_out = dy.shape[1] if d_out is None else d_out
        dt = _dtype_code(dy) if dtype is None else dtype
        self._check(self.lib.dfx_compose_bwd(self.ctx, dt, _ptr(dy), _ptr(g), float(s),
                                             _ptr(inner), _ptr(w_norm), rows, d_out, _ptr(d_lora),
                                             _ptr(d_base), _ptr(d_mag), _stream(stream)))

    def working_matmul(self, a, b, c, trans_a=False, trans_b=True, stream=None):
        """c = round(a' . b') with the reference's serial-k fp32 order, where a' = a^T if
        trans_a and b' = b^T if trans_b (row-major device tensors, no copies)."""
        M = a.shape[1] if trans_a else a.shape[0]
        K = a.shape[0] if trans_a else a.shape[1]
        N = b.shape[0] if trans_b else b.shape[1]
        sa_i, sa_k = (1, a.shape[1]) if trans_a else (a.shape[1], 1)
        sb_k, sb_j = (1, b.shape[1]) if trans_b else (b.shape[1], 1)
        self._check(self.lib.dfx_working_matmul(self.ctx, _dtype_code(a), _ptr(a), sa_i, sa_k,
                                                _ptr(b), sb_k, sb_j, M, N, K, _ptr(c),
                                                _stream(stream)))

    def set_sm_budget(self, sms: int):
        """Cap the SMs the norm GEMMs plan for (0 = all); see dfx_ctx_set_sm_budget."""
        self._check(self.lib.dfx_ctx_set_sm_budget(self.ctx, int(sms)))

    def lora_compose(self, mid, B, base, g, s, y=None, delta=None, inner=None, lora=None,
                     bias=None, stream=None):
        """Fused LoRA-up GEMM + compose + residual (device tensors)."""
        rows, r = mid.shape
        d_out = B.shape[0]
        self._check(self.lib.dfx_lora_compose(self.ctx, _dtype_code(mid), _ptr(mid), _ptr(B),
                                              _ptr(base), _ptr(g), float(s), _ptr(bias), rows,
                                              d_out, r, _ptr(y), _ptr(delta), _ptr(inner),
                                              _ptr(lora), _stream(stream)))

    def module_fwd_host(self, dtype, W, A, B, m, base, lora, s, d_out, d_in, r, rows,
                        chunk_size, delta, g):
        """Host (pinned CPU tensor) buffers in, host buffers out; blocking."""
        self._check(self.lib.dfx_module_fwd_host(self.ctx, dtype, _ptr(W), _ptr(A), _ptr(B),
                                                 _ptr(m), _ptr(base), _ptr(lora), float(s),
                                                 d_out, d_in, r, rows, chunk_size, _ptr(delta),
                                                 _ptr(g)))

    def module_train_host(self, dtype, W, A, B, m, base, lora, dy, s, d_out, d_in, r, rows,
                          chunk_size, delta, d_lora, d_base, d_mag, g):
        """Training step from host (pinned CPU tensor) buffers; blocking."""
        self._check(self.lib.dfx_module_train_host(self.ctx, dtype, _ptr(W), _ptr(A), _ptr(B),
                                                   _ptr(m), _ptr(base), _ptr(lora), _ptr(dy),
                                                   float(s), d_out, d_in, r, rows, chunk_size,
                                                   _ptr(delta), _ptr(d_lora), _ptr(d_base),
                                                   _ptr(d_mag), _ptr(g)))

    # ------------------------------------------------------------ profiling
    def profile(self, on: bool = True):
        self._check(self.lib.dfx_profile_enable(self.ctx, int(on)))

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms, min_ms, max_ms)}; synchronises and resets."""
        buf = C.create_string_buffer(1 << 16)
        self._check(self.lib.dfx_profile_report(self.ctx, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, tot, mn, mx = line.split()
            out[name] = (int(n), float(tot), float(mn), float(mx))
        return out

    # ----------------------------------------------------------------- misc
    def plan_chunks(self, d_out, d_in, budget=268435456):
        return plan_chunks(d_out, d_in, budget)

    def uses_tensor_cores(self, dtype, d_out, d_in, r) -> bool:
        return bool(self.lib.dfx_norm_uses_tensor_cores(dtype, d_out, d_in, r))


def plan_chunks(d_out, d_in, budget=268435456):
    """ChunkPlan (chunk_size, num_chunks) via the C ABI (host-only, no device needed)."""
    lib = load_library()
    cs, nc = C.c_uint64(), C.c_uint64()
    rc = lib.dfx_plan_chunks(d_out, d_in, budget, C.byref(cs), C.byref(nc))
    if rc != DFX_OK:
        raise DfxInvalidArgument(rc, lib.dfx_last_error().decode())
    return cs.value, nc.value
