"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module.  Two libraries are exposed with the same numpy-level surface:

* ``Oracle``    — oracle/liboracle.so, the C restatement (oracle/oracle.c);
* ``Reference`` — oracle/_ref/libdfx_ref.so, the reference's own sources compiled
  by oracle/Makefile (absent when the reference tree was never available).

All matrices are float32 numpy arrays whose values are representable in the
tagged dtype (0 fp32, 1 bf16, 2 fp16), mirroring the reference RealMatrix.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdfx_ref.so")

F32, BF16, F16, F64 = 0, 1, 2, 3
DTYPE_NAMES = {"fp32": F32, "bf16": BF16, "fp16": F16, "fp64": F64}

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_sz = C.c_size_t


def build() -> None:
    """Compile liboracle.so (and _ref when the reference tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_fp)


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


class Oracle:
    """oracle.c through ctypes (calls release the GIL, so threads run in parallel)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_round_to_dtype.restype = C.c_double
        L.orc_round_to_dtype.argtypes = [C.c_double, C.c_int]
        L.orc_plan_chunks.argtypes = [_sz, _sz, C.c_uint64, C.POINTER(_sz), C.POINTER(_sz)]
        L.orc_norm_terms.argtypes = [_fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _sz, _fp, _fp, _fp]
        L.orc_assemble.argtypes = [_fp, _fp, _fp, C.c_double, C.c_double, _sz, _fp]
        L.orc_row_norm.argtypes = [C.c_int, _fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _sz, _fp]
        L.orc_magnitude_scale.argtypes = [C.c_int, _dp, _fp, _sz, _fp]
        L.orc_compose_fwd.argtypes = [C.c_int, _fp, _fp, _fp, C.c_double, _sz, _sz, _fp, _fp]
        L.orc_naive_compose.argtypes = [C.c_int, _fp, _fp, _fp, C.c_double, _sz, _sz, _fp]
        L.orc_working_matmul_nt.argtypes = [C.c_int, _fp, _fp, _sz, _sz, _sz, _fp]
        L.orc_residual.argtypes = [C.c_int, _fp, _fp, _fp, _sz, _sz, _fp]
        L.orc_compose_bwd.argtypes = [C.c_int, _fp, _fp, C.c_double, _fp, _fp, _sz, _sz, C.c_int,
                                      _fp, _fp, _fp]
        L.orc_dense_row_norm_f64.argtypes = [_fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _dp]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_seeded_gaussian.argtypes = [_sz, C.c_uint64, C.c_int, _fp]
        L.orc_gaussian_fixture.argtypes = [_sz, C.c_double, C.c_double, C.c_uint64, C.c_int, _fp]
        L.orc_gaussian_vector.argtypes = [_sz, C.c_double, C.c_double, C.c_uint64, _dp]
        self.L = L

    # ---- numerics / planning
    def round_to_dtype(self, x: float, dtype: int) -> float:
        return self.L.orc_round_to_dtype(float(x), dtype)

    def plan_chunks(self, d_out, d_in, budget=268435456):
        cs, nc = _sz(), _sz()
        if self.L.orc_plan_chunks(d_out, d_in, budget, C.byref(cs), C.byref(nc)) != 0:
            raise ValueError("plan_chunks: invalid arguments")
        return cs.value, nc.value

    # ---- norm
    def norm_terms(self, w, a, b, s, chunk_size):
        d_out, d_in = w.shape
        r = a.shape[0]
        out = np.zeros((3, d_out), np.float32)
        rc = self.L.orc_norm_terms(_f(w), _f(a), _f(b), d_out, d_in, r, s, chunk_size,
                                   _f(out[0]), _f(out[1]), _f(out[2]))
        if rc != 0:
            raise ValueError("norm_terms: invalid arguments")
        return out[0], out[1], out[2]

    def assemble(self, base_sq, cross, ba_sq, two_s, s2):
        out = np.zeros(base_sq.shape[0], np.float32)
        self.L.orc_assemble(_f(base_sq), _f(cross), _f(ba_sq), two_s, s2, base_sq.shape[0], _f(out))
        return out

    def row_norm(self, dtype, w, a, b, s, chunk_size):
        d_out, d_in = w.shape
        out = np.zeros(d_out, np.float32)
        rc = self.L.orc_row_norm(dtype, _f(w), _f(a), _f(b), d_out, d_in, a.shape[0], s,
                                 chunk_size, _f(out))
        if rc != 0:
            raise ValueError("row_norm: invalid arguments")
        return out

    def magnitude_scale(self, dtype, m, w_norm):
        m = np.ascontiguousarray(m, np.float64)
        g = np.zeros(m.shape[0], np.float32)
        self.L.orc_magnitude_scale(dtype, _d(m), _f(w_norm), m.shape[0], _f(g))
        return g

    # ---- compose
    def compose_fwd(self, dtype, base, lora, g, s, need_inner=False):
        rows, d_out = base.shape
        delta = np.zeros_like(base)
        inner = np.zeros_like(base) if need_inner else None
        self.L.orc_compose_fwd(dtype, _f(base), _f(lora), _f(g), s, rows, d_out, _f(delta), _f(inner))
        return delta, inner

    def working_matmul_nt(self, dtype, a, bt):
        """round_dtype(a @ bt.T) with the reference's serial-k fp32 accumulation."""
        m, k = a.shape
        n = bt.shape[0]
        out = np.zeros((m, n), np.float32)
        self.L.orc_working_matmul_nt(dtype, _f(a), _f(bt), m, n, k, _f(out))
        return out

    def residual(self, dtype, base, delta, bias=None):
        rows, d_out = base.shape
        y = np.zeros_like(base)
        self.L.orc_residual(dtype, _f(base), _f(delta), _f(bias), rows, d_out, _f(y))
        return y

    def naive_compose(self, dtype, base, lora, g, s):
        rows, d_out = base.shape
        delta = np.zeros_like(base)
        self.L.orc_naive_compose(dtype, _f(base), _f(lora), _f(g), s, rows, d_out, _f(delta))
        return delta

    def compose_bwd(self, dtype, dy, g, s, inner=None, w_norm=None, mag_grad=False):
        rows, d_out = dy.shape
        d_lora = np.zeros_like(dy)
        d_base = np.zeros_like(dy)
        d_mag = np.zeros(d_out, np.float32) if mag_grad else None
        rc = self.L.orc_compose_bwd(dtype, _f(dy), _f(g), s, _f(inner), _f(w_norm), rows, d_out,
                                    int(mag_grad), _f(d_lora), _f(d_base), _f(d_mag))
        if rc != 0:
            raise ValueError("compose_backward: magnitude gradient requires inner")
        return d_lora, d_base, d_mag

    def dense_row_norm_f64(self, w, a, b, s):
        d_out, d_in = w.shape
        out = np.zeros(d_out, np.float64)
        self.L.orc_dense_row_norm_f64(_f(w), _f(a), _f(b), d_out, d_in, a.shape[0], s, _d(out))
        return out

    # ---- fixtures
    def derive_seed(self, base, index):
        return self.L.orc_derive_seed(base, index)

    def seeded_gaussian(self, rows, cols, seed, dtype=F32):
        out = np.zeros((rows, cols), np.float32)
        self.L.orc_seeded_gaussian(rows * cols, seed, dtype, _f(out))
        return out

    def gaussian_fixture(self, rows, cols, mean, stddev, seed, dtype=F32):
        out = np.zeros((rows, cols), np.float32)
        self.L.orc_gaussian_fixture(rows * cols, mean, stddev, seed, dtype, _f(out))
        return out

    def gaussian_vector(self, n, mean, stddev, seed):
        out = np.zeros(n, np.float64)
        self.L.orc_gaussian_vector(n, mean, stddev, seed, _d(out))
        return out


class Reference:
    """The reference's own code (oracle/_ref/libdfx_ref.so) through ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_plan_chunks.argtypes = [_sz, _sz, C.c_uint64, C.POINTER(_sz), C.POINTER(_sz)]
        L.ref_round_to_dtype.restype = C.c_double
        L.ref_round_to_dtype.argtypes = [C.c_double, C.c_int]
        L.ref_norm_terms.argtypes = [C.c_int, _fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _sz,
                                     _fp, _fp, _fp]
        L.ref_row_norm.argtypes = [C.c_int, _fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _sz, _dp]
        L.ref_assemble.argtypes = [_fp, _fp, _fp, C.c_double, C.c_double, _sz, _fp]
        L.ref_magnitude_scale.argtypes = [C.c_int, _dp, _dp, _sz, _dp]
        L.ref_compose.argtypes = [C.c_int, C.c_int, _fp, _fp, _dp, C.c_double, _sz, _sz, _fp, _fp]
        L.ref_compose_bwd.argtypes = [C.c_int, _fp, _dp, C.c_double, _fp, _dp, _sz, _sz, C.c_int,
                                      _fp, _fp, _dp]
        L.ref_layer_forward.argtypes = [C.c_int, _fp, _fp, _fp, _fp, C.c_double, _dp, _dp, _sz, _sz,
                                        _sz, _sz, _fp, _fp, _fp, _fp, _fp, _dp, _dp]
        L.ref_dense_row_norm_f64.argtypes = [_fp, _fp, _fp, _sz, _sz, _sz, C.c_double, _dp]
        L.ref_seeded_gaussian.argtypes = [_sz, _sz, C.c_uint64, C.c_int, _fp]
        L.ref_gaussian_fixture.argtypes = [_sz, _sz, C.c_double, C.c_double, C.c_uint64, C.c_int, _fp]
        L.ref_gaussian_vector.argtypes = [_sz, C.c_double, C.c_double, C.c_uint64, _dp]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_last_call_ns.restype = C.c_int64
        L.ref_last_call_ns.argtypes = []
        self.L = L

    def last_call_s(self) -> float:
        """Wall time of this thread's last reference call (RealMatrix packing excluded)."""
        return self.L.ref_last_call_ns() * 1e-9

    def round_to_dtype(self, x, dtype):
        return self.L.ref_round_to_dtype(float(x), dtype)

    def plan_chunks(self, d_out, d_in, budget=268435456):
        cs, nc = _sz(), _sz()
        if self.L.ref_plan_chunks(d_out, d_in, budget, C.byref(cs), C.byref(nc)) != 0:
            raise ValueError("plan_chunks: invalid arguments")
        return cs.value, nc.value

    def norm_terms(self, dtype, w, a, b, s, chunk_size):
        d_out, d_in = w.shape
        out = np.zeros((3, d_out), np.float32)
        if self.L.ref_norm_terms(dtype, _f(w), _f(a), _f(b), d_out, d_in, a.shape[0], s,
                                 chunk_size, _f(out[0]), _f(out[1]), _f(out[2])) != 0:
            raise ValueError("factored_norm_terms threw")
        return out[0], out[1], out[2]

    def row_norm(self, dtype, w, a, b, s, chunk_size):
        d_out, d_in = w.shape
        out = np.zeros(d_out, np.float64)
        if self.L.ref_row_norm(dtype, _f(w), _f(a), _f(b), d_out, d_in, a.shape[0], s,
                               chunk_size, _d(out)) != 0:
            raise ValueError("factored_row_norm threw")
        return out

    def assemble(self, base_sq, cross, ba_sq, two_s, s2):
        out = np.zeros(base_sq.shape[0], np.float32)
        self.L.ref_assemble(_f(base_sq), _f(cross), _f(ba_sq), two_s, s2, base_sq.shape[0], _f(out))
        return out

    def magnitude_scale(self, dtype, m, w_norm):
        m = np.ascontiguousarray(m, np.float64)
        wn = np.ascontiguousarray(w_norm, np.float64)
        g = np.zeros(m.shape[0], np.float64)
        if self.L.ref_magnitude_scale(dtype, _d(m), _d(wn), m.shape[0], _d(g)) != 0:
            raise ValueError("magnitude_scale threw")
        return g

    def compose(self, variant, dtype, base, lora, g, s, need_inner=False):
        rows, d_out = base.shape
        g = np.ascontiguousarray(g, np.float64)
        delta = np.zeros_like(base)
        inner = np.zeros_like(base) if need_inner else None
        if self.L.ref_compose(variant, dtype, _f(base), _f(lora), _d(g), s, rows, d_out,
                              _f(delta), _f(inner)) != 0:
            raise ValueError("compose threw")
        return delta, inner

    def compose_bwd(self, dtype, dy, g, s, inner=None, w_norm=None, mag_grad=False):
        rows, d_out = dy.shape
        g = np.ascontiguousarray(g, np.float64)
        wn = None if w_norm is None else np.ascontiguousarray(w_norm, np.float64)
        d_lora = np.zeros_like(dy)
        d_base = np.zeros_like(dy)
        d_mag = np.zeros(d_out, np.float64) if mag_grad else None
        if self.L.ref_compose_bwd(dtype, _f(dy), _d(g), s, _f(inner), _d(wn), rows, d_out,
                                  int(mag_grad), _f(d_lora), _f(d_base), _d(d_mag)) != 0:
            raise ValueError("compose_backward threw")
        return d_lora, d_base, d_mag

    def layer_forward(self, dtype, x, w, a, b, s, m, bias=None):
        """The reference's layer_forward; returns dict of y, lora_mid, base_out, lora_out,
        inner, g, w_norm."""
        rows, d_in = x.shape
        d_out, r = b.shape
        o = {k: np.zeros((rows, d_out), np.float32) for k in ("y", "base_out", "lora_out", "inner")}
        o["lora_mid"] = np.zeros((rows, r), np.float32)
        o["g"] = np.zeros(d_out, np.float64)
        o["w_norm"] = np.zeros(d_out, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        bias = None if bias is None else np.ascontiguousarray(bias, np.float64)
        if self.L.ref_layer_forward(dtype, _f(x), _f(w), _f(a), _f(b), s, _d(m), _d(bias), rows,
                                    d_in, d_out, r, _f(o["y"]), _f(o["lora_mid"]), _f(o["base_out"]),
                                    _f(o["lora_out"]), _f(o["inner"]), _d(o["g"]),
                                    _d(o["w_norm"])) != 0:
            raise ValueError("layer_forward threw")
        return o

    def dense_row_norm_f64(self, w, a, b, s):
        d_out, d_in = w.shape
        out = np.zeros(d_out, np.float64)
        self.L.ref_dense_row_norm_f64(_f(w), _f(a), _f(b), d_out, d_in, a.shape[0], s, _d(out))
        return out

    def seeded_gaussian(self, rows, cols, seed, dtype=F32):
        out = np.zeros((rows, cols), np.float32)
        self.L.ref_seeded_gaussian(rows, cols, seed, dtype, _f(out))
        return out

    def gaussian_fixture(self, rows, cols, mean, stddev, seed, dtype=F32):
        out = np.zeros((rows, cols), np.float32)
        self.L.ref_gaussian_fixture(rows, cols, mean, stddev, seed, dtype, _f(out))
        return out

    def gaussian_vector(self, n, mean, stddev, seed):
        out = np.zeros(n, np.float64)
        self.L.ref_gaussian_vector(n, mean, stddev, seed, _d(out))
        return out

    def derive_seed(self, base, index):
        return self.L.ref_derive_seed(base, index)


def reference_available() -> bool:
    return os.path.exists(REF_SO)
