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

__all__ = ["Dfx", "Comm", "build", "LIB_PATH", "DROPIN_PATH", "F32", "BF16", "F16", "DfxError"]

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
    "dfx_norm_adapter": (_int, [_vp, _int, _vp, _vp, _i64, _i64, _i64, _int, _vp, _vp]),
    "dfx_row_norm_ba": (_int, [_vp, _int, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _i64, _vp, _vp,
                               _int, _vp, _vp, _vp, _vp]),
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
    "dfx_comm_create": (_int, [_vp, _int, _int, _i64, C.POINTER(_vp)]),
    "dfx_comm_destroy": (None, [_vp]),
    "dfx_comm_buffer": (_vp, [_vp]),
    "dfx_comm_base": (_vp, [_vp]),
    "dfx_comm_ipc_handle": (_int, [_vp, _vp]),
    "dfx_comm_open": (_int, [_vp, _vp]),
    "dfx_comm_set_peers": (_int, [_vp, C.POINTER(_vp)]),
    "dfx_norm_allreduce": (_int, [_vp, _vp, _i64, _vp]),
    "dfx_comm_status": (_int, [_vp, C.POINTER(_int)]),
}

IPC_HANDLE_BYTES = 64

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


def _stream(stream, device=None):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream(device).cuda_stream


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

    def _s(self, stream):
        """The caller's stream, or torch's current stream of THIS context's device."""
        return _stream(stream, self.device)

    def _t(self, name, t, dtype=None, shape=None, min_numel=None):
        """Validate a tensor argument before its pointer crosses the C ABI: on this context's
        device, contiguous (the kernels assume dense row-major; the reference throws
        std::invalid_argument on non-contiguous input, compose.cpp:72-75), of the expected
        dtype and shape.  Raw integer pointers are passed through unchecked."""
        if t is None or isinstance(t, int):
            return
        if not t.is_cuda or t.device.index != self.device:
            raise DfxInvalidArgument(DFX_EINVAL, f"{name}: tensor on {t.device}, context on "
                                                 f"cuda:{self.device}")
        if not t.is_contiguous():
            raise DfxInvalidArgument(DFX_EINVAL, f"{name}: non-contiguous tensor (call "
                                                 f".contiguous() first)")
        if dtype is not None and t.dtype != dtype:
            raise DfxInvalidArgument(DFX_EINVAL, f"{name}: dtype {t.dtype}, expected {dtype}")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise DfxInvalidArgument(DFX_EINVAL, f"{name}: shape {tuple(t.shape)}, expected "
                                                 f"{tuple(shape)}")
        if min_numel is not None and t.numel() < min_numel:
            raise DfxInvalidArgument(DFX_EINVAL, f"{name}: {t.numel()} elements, need "
                                                 f"{min_numel}")

    def _norm_operands(self, W, A, B):
        """Shapes/dtypes of W [d_out, d_in], A [r, d_in], B [d_out, r] as the reference checks
        them (factored_norm.cpp:11-23); returns (d_out, d_in, r)."""
        d_out, d_in = W.shape
        r = A.shape[0]
        self._t("W", W)
        self._t("A", A, dtype=W.dtype, shape=(r, d_in))
        self._t("B", B, dtype=W.dtype, shape=(d_out, r))
        return d_out, d_in, r

    def _vec(self, name, t, n):
        import torch
        self._t(name, t, dtype=torch.float32, min_numel=n)

    @property
    def launches(self) -> int:
        return int(self.lib.dfx_ctx_launches(self.ctx))

    # ----------------------------------------------------------------- norm
    def norm_terms(self, W, A, B, s, chunk_size, base_sq, cross, ba_sq, stream=None):
        d_out, d_in, r = self._norm_operands(W, A, B)
        for nm, v in (("base_sq", base_sq), ("cross", cross), ("ba_sq", ba_sq)):
            self._vec(nm, v, d_out)
        self._check(self.lib.dfx_norm_terms(self.ctx, _dtype_code(W), _ptr(W), _ptr(A), _ptr(B),
                                            d_out, d_in, r, float(s), int(chunk_size),
                                            _ptr(base_sq), _ptr(cross), _ptr(ba_sq),
                                            self._s(stream)))

    def row_norm(self, W, A, B, s, chunk_size, w_norm, m=None, g=None, terms=None,
                 mag_dtype=None, stream=None):
        d_out, d_in, r = self._norm_operands(W, A, B)
        self._vec("w_norm", w_norm, d_out)
        self._vec("m", m, d_out)
        self._vec("g", g, d_out)
        self._vec("terms", terms, 3 * d_out)
        dt = _dtype_code(W)
        self._check(self.lib.dfx_row_norm(self.ctx, dt, _ptr(W), _ptr(A), _ptr(B), d_out, d_in, r,
                                          float(s), int(chunk_size), _ptr(m),
                                          dt if mag_dtype is None else mag_dtype, _ptr(w_norm),
                                          _ptr(g), _ptr(terms), self._s(stream)))

    def norm_plan(self, d_out, d_in, r, chunk_size, dtype=BF16):
        """(u_sms, side_sms, strategy) of the tensor-core norm under the current SM budget."""
        u, sd, st = C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.dfx_norm_plan(self.ctx, dtype, d_out, d_in, r, int(chunk_size),
                                           C.byref(u), C.byref(sd), C.byref(st)))
        return u.value, sd.value, st.value

    def norm_adapter(self, A, B, d_out, ba_sq, sms=0, stream=None):
        """dfx_norm_adapter: ba_sq = rowquad(B, A A^T) [d_out] fp32 (the adapter-only part of the
        factored norm, for pipelined stacks; bf16 / fp16); sms > 0 caps the SMs it plans for."""
        r, d_in = A.shape
        self._vec("ba_sq", ba_sq, d_out)
        self._check(self.lib.dfx_norm_adapter(self.ctx, _dtype_code(A), _ptr(A), _ptr(B), d_out, d_in,
                                              r, int(sms), _ptr(ba_sq), self._s(stream)))

    def row_norm_ba(self, W, A, B, s, chunk_size, ba_sq, w_norm, m=None, g=None, terms=None,
                    mag_dtype=None, stream=None):
        """dfx_row_norm_ba: the W part of the norm, finished with a ba_sq from norm_adapter."""
        d_out, d_in, r = self._norm_operands(W, A, B)
        self._vec("ba_sq", ba_sq, d_out)
        self._vec("w_norm", w_norm, d_out)
        dt = _dtype_code(W)
        md = dt if mag_dtype is None else mag_dtype
        self._check(self.lib.dfx_row_norm_ba(self.ctx, dt, _ptr(W), _ptr(A), _ptr(B), d_out, d_in, r,
                                             float(s), int(chunk_size), _ptr(ba_sq), _ptr(m), md,
                                             _ptr(w_norm), _ptr(g), _ptr(terms), self._s(stream)))

    def row_norm_cached(self, W, A, B, s, chunk_size, base_sq_cache, w_norm, refresh=False,
                        m=None, g=None, mag_dtype=None, stream=None):
        """Opt-in cached ||W||^2_row for a frozen W (dfx_row_norm_cached)."""
        d_out, d_in, r = self._norm_operands(W, A, B)
        for nm, v in (("base_sq_cache", base_sq_cache), ("w_norm", w_norm), ("m", m), ("g", g)):
            self._vec(nm, v, d_out)
        dt = _dtype_code(W)
        self._check(self.lib.dfx_row_norm_cached(
            self.ctx, dt, _ptr(W), _ptr(A), _ptr(B), d_out, d_in, r, float(s), int(chunk_size),
            _ptr(base_sq_cache), 1 if refresh else 0, _ptr(m),
            dt if mag_dtype is None else mag_dtype, _ptr(w_norm), _ptr(g), self._s(stream)))

    def norm_partial(self, W_k, A_k, B, chunk_size, gram, base_sq, cross, stream=None):
        """d_in-split step 1: this rank's K-slice terms (sum them over ranks).  W_k must be a
        contiguous copy of the rank's columns (a column slice W[:, k0:k1] is not)."""
        d_out, d_in_k, r = self._norm_operands(W_k, A_k, B)
        self._vec("gram", gram, r * r)
        self._vec("base_sq", base_sq, d_out)
        self._vec("cross", cross, d_out)
        self._check(self.lib.dfx_norm_partial(self.ctx, _dtype_code(W_k), _ptr(W_k), _ptr(A_k),
                                              _ptr(B), d_out, d_in_k, r, int(chunk_size),
                                              _ptr(gram), _ptr(base_sq), _ptr(cross),
                                              self._s(stream)))

    def norm_finish(self, B, gram, base_sq, cross, s, w_norm, m=None, g=None, terms=None,
                    mag_dtype=None, stream=None):
        """d_in-split step 2 from the reduced {gram, base_sq, cross}."""
        d_out, r = B.shape
        self._t("B", B)
        self._vec("gram", gram, r * r)
        for nm, v in (("base_sq", base_sq), ("cross", cross), ("w_norm", w_norm), ("m", m),
                      ("g", g)):
            self._vec(nm, v, d_out)
        self._vec("terms", terms, 3 * d_out)
        dt = _dtype_code(B)
        self._check(self.lib.dfx_norm_finish(self.ctx, dt, _ptr(B), _ptr(gram), _ptr(base_sq),
                                             _ptr(cross), d_out, r, float(s), _ptr(m),
                                             dt if mag_dtype is None else mag_dtype, _ptr(w_norm),
                                             _ptr(g), _ptr(terms), self._s(stream)))

    def assemble(self, base_sq, cross, ba_sq, two_s, s2, out, round_to=F32, n=None,
                 stream=None):
        n = base_sq.shape[0] if n is None else n
        self._check(self.lib.dfx_assemble_norm(self.ctx, _ptr(base_sq), _ptr(cross), _ptr(ba_sq),
                                               float(two_s), float(s2), n, round_to, _ptr(out),
                                               self._s(stream)))

    def magnitude_scale(self, dtype, m, w_norm, g, n=None, stream=None):
        n = m.shape[0] if n is None else n
        self._check(self.lib.dfx_magnitude_scale(self.ctx, dtype, _ptr(m), _ptr(w_norm), n,
                                                 _ptr(g), self._s(stream)))

    # -------------------------------------------------------------- compose
    def compose_fwd(self, base, lora, g, s, delta, inner=None, stream=None, dtype=None,
                    rows=None, d_out=None):
        rows = base.shape[0] if rows is None else rows
        d_out = base.shape[1] if d_out is None else d_out
        if not isinstance(base, int):
            self._t("base", base)
            for nm, v in (("lora", lora), ("delta", delta), ("inner", inner)):
                self._t(nm, v, dtype=base.dtype, min_numel=rows * d_out)
            self._vec("g", g, d_out)
        dt = _dtype_code(base) if dtype is None else dtype
        self._check(self.lib.dfx_compose_fwd(self.ctx, dt, _ptr(base), _ptr(lora), _ptr(g),
                                             float(s), rows, d_out, _ptr(delta), _ptr(inner),
                                             self._s(stream)))

    def compose_bwd(self, dy, g, s, d_lora, d_base, inner=None, w_norm=None, d_mag=None,
                    stream=None, dtype=None, rows=None, d_out=None):
        rows = dy.shape[0] if rows is None else rows
        d_out = dy.shape[1] if d_out is None else d_out
        if not isinstance(dy, int):
            self._t("dy", dy)
            for nm, v in (("d_lora", d_lora), ("d_base", d_base), ("inner", inner)):
                self._t(nm, v, dtype=dy.dtype, min_numel=rows * d_out)
            for nm, v in (("g", g), ("w_norm", w_norm), ("d_mag", d_mag)):
                self._vec(nm, v, d_out)
        dt = _dtype_code(dy) if dtype is None else dtype
        self._check(self.lib.dfx_compose_bwd(self.ctx, dt, _ptr(dy), _ptr(g), float(s),
                                             _ptr(inner), _ptr(w_norm), rows, d_out, _ptr(d_lora),
                                             _ptr(d_base), _ptr(d_mag), self._s(stream)))

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
                                                self._s(stream)))

    def set_sm_budget(self, sms: int):
        """Cap the SMs the norm GEMMs plan for (0 = all); see dfx_ctx_set_sm_budget."""
        self._check(self.lib.dfx_ctx_set_sm_budget(self.ctx, int(sms)))
        self._budget = int(sms)

    def get_sm_budget(self) -> int:
        """The budget last set through this binding (0 = all SMs)."""
        return getattr(self, "_budget", 0)

    def lora_compose(self, mid, B, base, g, s, y=None, delta=None, inner=None, lora=None,
                     bias=None, stream=None):
        """Fused LoRA-up GEMM + compose + residual (device tensors)."""
        rows, r = mid.shape
        d_out = B.shape[0]
        self._t("mid", mid)
        self._t("B", B, dtype=mid.dtype, shape=(d_out, r))
        self._t("base", base, dtype=mid.dtype, shape=(rows, d_out))
        for nm, v in (("y", y), ("delta", delta), ("inner", inner), ("lora", lora)):
            self._t(nm, v, dtype=mid.dtype, shape=(rows, d_out))
        self._vec("g", g, d_out)
        self._vec("bias", bias, d_out)
        self._check(self.lib.dfx_lora_compose(self.ctx, _dtype_code(mid), _ptr(mid), _ptr(B),
                                              _ptr(base), _ptr(g), float(s), _ptr(bias), rows,
                                              d_out, r, _ptr(y), _ptr(delta), _ptr(inner),
                                              _ptr(lora), self._s(stream)))

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

    # ------------------------------------------------------- symmetric all-reduce
    def comm(self, rank: int, world: int, count: int) -> "Comm":
        """A symmetric-memory all-reduce endpoint on this context (dfx_comm_create)."""
        return Comm(self, rank, world, count)

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


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (torch.as_tensor reads it;
    the owner keeps the memory alive)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class Comm:
    """One rank's endpoint of the symmetric-memory all-reduce (include/dfx.h, dfx_comm_*):
    buffer() is this rank's symmetric data region as a float32 CUDA tensor (write the partial
    terms there), ipc_handle()/open(handles) or set_peers(bases) map the peers, and
    all_reduce(out) writes the rank-order sum of every rank's buffer into `out`."""

    def __init__(self, dfx: "Dfx", rank: int, world: int, count: int):
        self.dfx, self.lib = dfx, dfx.lib
        self.rank, self.world, self.count = rank, world, count
        h = _vp()
        dfx._check(self.lib.dfx_comm_create(dfx.ctx, rank, world, count, C.byref(h)))
        self.h = h

    def buffer(self):
        import torch
        ptr = self.lib.dfx_comm_buffer(self.h)
        return torch.as_tensor(_CudaArray(ptr, self.count), device=f"cuda:{self.dfx.device}")

    def base(self) -> int:
        return int(self.lib.dfx_comm_base(self.h))

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        self.dfx._check(self.lib.dfx_comm_ipc_handle(self.h, buf))
        return buf.raw

    def open(self, handles):
        """handles: list of `world` IPC handles (bytes) in rank order."""
        blob = b"".join(handles)
        self.dfx._check(self.lib.dfx_comm_open(self.h, C.c_char_p(blob)))

    def set_peers(self, bases):
        arr = (_vp * self.world)(*bases)
        self.dfx._check(self.lib.dfx_comm_set_peers(self.h, arr))

    def all_reduce(self, out, count=None, stream=None):
        n = self.count if count is None else count
        self.dfx._vec("out", out, n)
        self.dfx._check(self.lib.dfx_norm_allreduce(self.h, _ptr(out), n, self.dfx._s(stream)))

    def status(self) -> int:
        """1 when a barrier spin timed out since creation (a peer never arrived), else 0."""
        t = _int()
        self.dfx._check(self.lib.dfx_comm_status(self.h, C.byref(t)))
        return t.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.dfx_comm_destroy(self.h)
            self.h = None
