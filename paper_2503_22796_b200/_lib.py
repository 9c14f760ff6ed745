"""ctypes binding of the C-ABI in include/dfa2c.h (libdfa2_b200.so, in-tree).

The product path has no fallback: if the native library is missing or a
call fails, an exception mirroring the reference's error taxonomy
(/root/reference/proj/include/dfa2/errors.hpp:8-45) is raised.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_uint8, c_uint32, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFA2_LIB") or os.path.join(HERE, "libdfa2_b200.so")  # DFA2_LIB: A/B builds


class Dfa2Error(RuntimeError):
    """Base of the mapped status codes."""


class ShapeError(Dfa2Error, ValueError):
    """dfa2::ShapeError (a std::invalid_argument in the reference)."""


class NonFiniteError(Dfa2Error):
    pass


class FullyMaskedRowError(Dfa2Error):
    pass


class CacheMissError(Dfa2Error):
    pass


class DegenerateReferenceError(Dfa2Error):
    pass


class PlanValidationError(Dfa2Error):
    pass


class IoError(Dfa2Error):
    pass


class OracleError(Dfa2Error):
    pass


class CudaError(Dfa2Error):
    pass


class UnsupportedError(Dfa2Error):
    pass


_ERRORS = {
    1: ShapeError,
    2: NonFiniteError,
    3: FullyMaskedRowError,
    4: CacheMissError,
    5: DegenerateReferenceError,
    6: PlanValidationError,
    7: IoError,
    8: OracleError,
    9: CudaError,
    10: UnsupportedError,
}


class Dims(ctypes.Structure):
    """dfa2c_dims (AttentionDims, inc/tensor.hpp:56-72)."""

    _fields_ = [
        ("n_heads", c_int64),
        ("head_dim", c_int64),
        ("n_visual", c_int64),
        ("n_text", c_int64),
        ("order", c_int32),
    ]


# name -> (restype, argtypes)
class PlanHeader(ctypes.Structure):
    """dfa2c_plan_header."""
    _fields_ = [("n_timesteps", c_int64), ("n_layers", c_int64), ("n_heads", c_int64), ("head_dim", c_int64),
                ("n_visual", c_int64), ("n_text", c_int64), ("block_size", c_int64), ("delta", c_double),
                ("coeff", c_double), ("n_window_set", c_int64), ("digest_len", c_int64)]


_SIGS = {
    "dfa2c_last_error": (c_char_p, []),
    "dfa2c_version": (c_char_p, []),
    "dfa2c_launch_count": (c_int64, []),
    "dfa2c_debug_set_trace": (None, [c_void_p]),
    "dfa2c_debug_schedule": (c_int32, [POINTER(c_double), c_int64, c_int32, c_int32, POINTER(c_int32),
                                       POINTER(c_double)]),
    "dfa2c_arrow_mask": (c_int32, [POINTER(Dims), c_int64, c_int64, POINTER(c_uint8), POINTER(c_int64)]),
    "dfa2c_mask_stats": (c_int32, [POINTER(c_uint8), c_int64, c_int64, c_int64, POINTER(c_int64),
                                   POINTER(c_int64), POINTER(c_double)]),
    "dfa2c_dense_flops": (c_int64, [c_int64, c_int64]),
    "dfa2c_kv_tile_keys": (c_int64, []),
    "dfa2c_plan_flops": (c_int32, [POINTER(Dims), c_int64, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    "dfa2c_plan_aggregate": (c_int32, [POINTER(Dims), c_int64, c_int64, c_int64, POINTER(c_int32),
                                       POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_double)]),
    "dfa2c_tile_set": (c_int32, [POINTER(Dims), c_int64, c_int32, c_int64, POINTER(c_int64),
                                 POINTER(c_uint32), POINTER(c_int64)]),
    "dfa2c_cache_create": (c_int32, [c_int64, c_int64, c_int64, c_int64, c_int64, POINTER(c_void_p)]),
    "dfa2c_cache_destroy": (c_int32, [c_void_p]),
    "dfa2c_cache_has": (c_int32, [c_void_p, c_int64, c_int64, POINTER(c_int32)]),
    "dfa2c_cache_produced_at": (c_int32, [c_void_p, c_int64, c_int64, POINTER(c_int64)]),
    "dfa2c_cache_staleness": (c_int32, [c_void_p, c_int64, c_int64, c_int64, POINTER(c_int64)]),
    "dfa2c_cache_store": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    "dfa2c_cache_fetch": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "dfa2c_cache_clear": (c_int32, [c_void_p]),
    "dfa2c_cache_size": (c_int32, [c_void_p, POINTER(c_int64)]),
    "dfa2c_cache_bytes": (c_int32, [c_void_p, POINTER(c_int64)]),
    "dfa2c_mha_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(Dims), c_int64,
                                    POINTER(c_int32), POINTER(c_int64), c_void_p, c_int64, c_int64,
                                    c_void_p, c_void_p]),
    "dfa2c_mha_forward_host": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(Dims), c_int64,
                                         POINTER(c_int32), POINTER(c_int64), c_void_p, c_int64, c_int64,
                                         c_void_p, c_void_p]),
    "dfa2c_sparse_attention_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                                 c_int64, POINTER(c_uint8), c_int64, c_void_p]),
    "dfa2c_dense_attention_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                                c_int64, c_void_p]),
    "dfa2c_mha_forward_sharded": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(Dims), c_int64,
                                            POINTER(c_int32), POINTER(c_int64), c_void_p, c_int64, c_int64,
                                            c_void_p, c_int32, c_int32, c_void_p, POINTER(c_int64), c_void_p]),
    "dfa2c_mha_forward_sharded_p2p": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(Dims), c_int64,
                                                POINTER(c_int32), POINTER(c_int64), c_void_p, c_int64, c_int64,
                                                POINTER(c_void_p), c_int32, c_int32, POINTER(c_int64), c_void_p]),
    "dfa2c_ipc_handle": (c_int32, [c_void_p, c_char_p, POINTER(c_int64)]),
    "dfa2c_ipc_open": (c_int32, [c_char_p, c_int64, POINTER(c_void_p)]),
    "dfa2c_ipc_close": (c_int32, [c_void_p, c_int64]),
    "dfa2c_shard_rows": (c_int32, [c_int64, POINTER(Dims), c_int64, POINTER(c_int32), POINTER(c_int64), c_int32,
                                   POINTER(c_int64)]),
    "dfa2c_shard_commit": (c_int32, [c_int64, POINTER(Dims), POINTER(c_int32), c_void_p, c_int64, POINTER(c_int64),
                                     c_int32, c_int32, c_void_p, c_void_p]),
    "dfa2c_nccl_available": (c_int32, []),
    "dfa2c_nccl_unique_id": (c_int32, [c_char_p]),
    "dfa2c_nccl_comm_init": (c_int32, [c_char_p, c_int32, c_int32, POINTER(c_void_p)]),
    "dfa2c_nccl_comm_destroy": (c_int32, [c_void_p]),
    "dfa2c_allgather_rows": (c_int32, [c_void_p, c_void_p, POINTER(c_int64), c_int32, c_int64, c_void_p]),
    "dfa2c_workload_create": (c_int32, [POINTER(Dims), c_int64, c_int64, ctypes.c_uint64, POINTER(c_void_p)]),
    "dfa2c_workload_destroy": (c_int32, [c_void_p]),
    "dfa2c_workload_profile": (c_int32, [c_void_p, c_int64, c_int64, POINTER(c_double), POINTER(c_double)]),
    "dfa2c_workload_slot": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dfa2c_attention_reference": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_int64,
                                            c_int64, POINTER(c_uint8), c_int64, c_void_p]),
    "dfa2c_rse": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_int32, POINTER(c_double),
                            c_void_p]),
    "dfa2c_rse_async": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_int32, c_void_p,
                                  c_void_p]),
    "dfa2c_plan_to_json": (c_int32, [POINTER(PlanHeader), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64),
                                     c_char_p, c_char_p, c_int64, POINTER(c_int64)]),
    "dfa2c_plan_from_json": (c_int32, [c_char_p, c_int64, POINTER(PlanHeader), POINTER(c_int32), POINTER(c_int64),
                                       POINTER(c_int64), c_char_p, c_int64]),
    "dfa2c_fnv1a_hex": (c_int32, [c_char_p, c_int64, c_char_p]),
    "dfa2c_set_split_kv": (c_int32, [c_int32]),
    "dfa2c_set_influence_fused": (c_int32, [c_int32]),
    "dfa2c_release_cached_memory": (c_int32, []),
    "dfa2c_influence_fused_enabled": (c_int32, []),
    "dfa2c_convert": (c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_int64, c_void_p]),
    "dfa2c_selection_cap": (c_double, [c_double, c_int64, c_double]),
    "dfa2c_plan_solve": (c_int32, [c_int64, c_int64, POINTER(c_double), c_double, POINTER(c_double), c_double,
                                   c_double, c_int32, POINTER(c_int64), POINTER(c_double), POINTER(c_double),
                                   POINTER(c_int64)]),
    "dfa2c_plan_lp_bound": (c_int32, [c_int64, c_int64, POINTER(c_double), c_double, POINTER(c_double), c_double,
                                      c_double, POINTER(c_double)]),
    "dfa2c_analytic_costs": (c_int32, [POINTER(Dims), c_int64, POINTER(c_int32), POINTER(c_int64), c_int64,
                                       POINTER(c_double), POINTER(c_double)]),
    "dfa2c_influence_for_layer": (c_int32, [c_void_p, c_void_p, c_void_p, POINTER(Dims), c_int64,
                                            POINTER(c_int64), c_int64, c_int32, c_void_p, c_int64, c_int64,
                                            c_int32, POINTER(c_double), c_void_p, c_void_p, POINTER(c_int64),
                                            c_void_p]),
    "dfa2c_influence_for_layer_async": (c_int32, [c_void_p, c_void_p, c_void_p, POINTER(Dims), c_int64,
                                                  POINTER(c_int64), c_int64, c_int32, c_void_p, c_int64, c_int64,
                                                  c_int32, POINTER(c_double), POINTER(c_uint8), c_void_p, c_void_p,
                                                  POINTER(c_int64), c_void_p]),
    "dfa2c_influence_finalize": (c_int32, [POINTER(c_double), POINTER(c_uint8), c_int64, c_int64,
                                           POINTER(c_double)]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libdfa2_b200.so (raising loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2503_22796_b200.build` "
                "(there is no CPU fallback for the attention path)")
        L = ctypes.CDLL(LIB_PATH)
        ab_build = os.path.abspath(LIB_PATH) != os.path.join(HERE, "libdfa2_b200.so")
        for name, (res, args) in _SIGS.items():
            if ab_build and not hasattr(L, name):
                continue  # an older A/B build without a newer entry point
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().dfa2c_last_error().decode(errors="replace")
        raise _ERRORS.get(status, Dfa2Error)(msg)


def exported_symbols():
    return list(_SIGS)
