"""TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes bindings for
  * liboracle.so        — the plain-C restatement (oracle.c), and
  * _ref/libdfa2ref.so  — the UNMODIFIED reference compiled in place
                          (Makefile `ref`), used to pin the restatement and as
                          the CPU baseline.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint8, c_uint16, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdfa2ref.so")
REF_SRC = "/root/reference/proj/src"


def build(ref: bool = True) -> None:
    """Builds liboracle.so, and oracle/_ref when the reference sources exist."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "-j8", "ref"], check=True)


def build_reftests() -> None:
    """Compiles the reference's own unit suites against the drop-in headers
    and the built libdfa2_b200.so (oracle/_ref/tests/; needs /root/reference
    and the product library)."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "-j8", "reftests"], check=True)


_P = lambda t: POINTER(t)  # noqa: E731
_orc = None
_ref = None


def orc() -> ctypes.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_arrow_mask.restype = c_int64
        L.orc_arrow_mask.argtypes = [c_int64, c_int64, c_int, c_int64, c_int64, _P(c_uint8)]
        L.orc_active_positions.restype = c_int64
        L.orc_active_positions.argtypes = [_P(c_uint8), c_int64, c_int64]
        L.orc_plan_flops.restype = c_int64
        L.orc_plan_flops.argtypes = [c_int64, c_int64, c_int64, c_int64, c_int, c_int64, _P(c_int32), _P(c_int64)]
        L.orc_sparse_forward_f32.restype = c_int
        L.orc_sparse_forward_f32.argtypes = [_P(c_float)] * 4 + [c_int64, c_int64, _P(c_uint8), c_int64]
        L.orc_attention_rows_f64.restype = c_int
        L.orc_attention_rows_f64.argtypes = [_P(c_float)] * 3 + [c_int64, c_int64, _P(c_uint8), c_int64,
                                                                 _P(c_int64), c_int64, _P(c_double)]
        L.orc_rse_f32.restype = c_int
        L.orc_rse_f32.argtypes = [_P(c_float), _P(c_float), c_int64, c_int, _P(c_double)]
        L.orc_rse_bf16.restype = c_int
        L.orc_rse_bf16.argtypes = [_P(c_uint16), _P(c_uint16), c_int64, c_int, _P(c_double)]
        L.orc_round_bf16.restype = None
        L.orc_round_bf16.argtypes = [_P(c_float), c_int64]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> ctypes.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build(ref=True)
        L = ctypes.CDLL(REF_SO)
        L.ref_last_error.restype = c_char_p
        sig = {
            "ref_arrow_mask": [c_int64] * 4 + [c_int, c_int64, c_int64, _P(c_uint8), _P(c_int64)],
            "ref_mask_stats": [_P(c_uint8), c_int64, c_int64, c_int64, _P(c_int64), _P(c_int64), _P(c_double)],
            "ref_plan_flops": [c_int64] * 4 + [c_int, c_int64, _P(c_int32), _P(c_int64), _P(c_int64)],
            "ref_sparse_attention_forward": [_P(c_float)] * 4 + [c_int64, c_int64, _P(c_uint8), c_int64, c_int],
            "ref_dense_tiled_attention": [_P(c_float)] * 4 + [c_int64, c_int64, c_int64, c_int],
            "ref_attention_reference_f64": [_P(c_double)] * 4 + [c_int64, c_int64, c_int64, _P(c_uint8), c_int64],
            "ref_attention_reference_f32": [_P(c_float)] * 4 + [c_int64, c_int64, c_int64, _P(c_uint8), c_int64],
            "ref_cache_store": [c_void_p, c_int64, c_int64, _P(c_float), c_int64, c_int64, c_int64],
            "ref_cache_has": [c_void_p, c_int64, c_int64],
            "ref_cache_produced_at": [c_void_p, c_int64, c_int64, _P(c_int64)],
            "ref_cache_fetch": [c_void_p, c_int64, c_int64, _P(c_float), c_int64],
            "ref_multi_strategy_attention": [_P(c_float)] * 3 + [c_int64] * 4 + [c_int, _P(c_int32), _P(c_int64),
                                                                                  c_void_p, c_int64, c_int64,
                                                                                  c_int64, _P(c_float)],
            "ref_rse": [_P(c_float), _P(c_float), c_int64, c_int, _P(c_double)],
            "ref_influence_for_layer": [_P(c_float)] * 3 + [c_int64] * 4 + [c_int, _P(c_int64), c_int64, c_int,
                                                                             c_void_p, c_int64, c_int64, c_int64,
                                                                             c_int, _P(c_double), _P(c_float),
                                                                             _P(c_float), _P(c_int64)],
            "ref_generate": [c_int64] * 4 + [c_int, c_int64, c_int64, c_int64, c_uint64, _P(c_float), _P(c_float),
                                             _P(c_float)],
            "ref_calibrate_model": [c_int64] * 4 + [c_int, c_int64, c_int64, c_int64, c_uint64, _P(c_int64), c_int64,
                                                    c_int, c_double, c_double, _P(c_int32), _P(c_int64), _P(c_double),
                                                    _P(c_double)],
            "ref_plan_aggregate": [c_int64] * 4 + [c_int, c_int64, c_int64, c_int64, _P(c_int32), _P(c_int64),
                                                   _P(c_int64), _P(c_int64), _P(c_double)],
            "ref_layer_sample": [_P(c_float)] * 5 + [c_int64] * 4 + [c_int, c_int64, _P(c_int32), _P(c_int64),
                                                                      _P(c_int64), c_int64],
            "ref_plan_to_json": [c_int64] * 7 + [c_double, c_double, _P(c_int64), c_int64, _P(c_int32), _P(c_int64),
                                                 c_char_p, c_char_p, c_int64, _P(c_int64)],
            "ref_plan_from_json": [c_char_p, c_int64, _P(c_int32), _P(c_int64), _P(c_int64)],
            "ref_plan_solve": [c_int64, c_int64, _P(c_double), c_double, _P(c_double), c_double, c_double, c_int,
                               _P(c_int64), _P(c_double), _P(c_double), _P(c_double)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c_int
        L.ref_cache_create.restype = c_void_p
        L.ref_cache_create.argtypes = []
        L.ref_cache_destroy.restype = None
        L.ref_cache_destroy.argtypes = [c_void_p]
        L.ref_dense_flops.restype = c_int64
        L.ref_dense_flops.argtypes = [c_int64, c_int64]
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


def ref_check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, ref().ref_last_error().decode(errors="replace"))


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(POINTER(t))


# ------------------------------------------------------------------ helpers
def round_bf16(x: np.ndarray) -> np.ndarray:
    """f32 -> bf16 -> f32 (round to nearest even), as torch does."""
    y = np.ascontiguousarray(x, dtype=np.float32).copy()
    orc().orc_round_bf16(ptr(y, c_float), y.size)
    return y


def arrow_mask(nv, nt, order, B, w) -> np.ndarray:
    nb = orc().orc_arrow_mask(nv, nt, order, B, w, None)
    m = np.zeros(nb * nb, np.uint8)
    orc().orc_arrow_mask(nv, nt, order, B, w, ptr(m, c_uint8))
    return m


def attention_rows_f64(q, k, v, mask=None, B=1, rows=None) -> np.ndarray:
    """Masked two-pass attention in f64 for one head (q/k/v f32 [N, d])."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    n, d = q.shape
    r = None if rows is None else np.ascontiguousarray(rows, np.int64)
    nr = n if r is None else r.size
    out = np.zeros((nr, d), np.float64)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    rc = orc().orc_attention_rows_f64(ptr(q, c_float), ptr(k, c_float), ptr(v, c_float), n, d,
                                      None if m is None else ptr(m, c_uint8), B,
                                      None if r is None else ptr(r, c_int64), nr, ptr(out, c_double))
    if rc:
        raise RuntimeError(f"oracle attention failed ({rc})")
    return out


def rse_f32(y_m, y_o, mode=0) -> float:
    a = np.ascontiguousarray(y_m, np.float32).ravel()
    b = np.ascontiguousarray(y_o, np.float32).ravel()
    out = c_double()
    rc = orc().orc_rse_f32(ptr(a, c_float), ptr(b, c_float), a.size, mode, ctypes.byref(out))
    if rc:
        raise RuntimeError(f"oracle rse failed ({rc})")
    return out.value


def gaussian(shape, seed) -> np.ndarray:
    """Seeded N(0,1) f32 (numpy PCG64; the synthetic-input generator of the tests/bench)."""
    return np.random.default_rng(seed).standard_normal(shape, dtype=np.float32)
