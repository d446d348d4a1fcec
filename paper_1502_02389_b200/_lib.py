"""ctypes loader for liblift.so — the C ABI declared in include/lift.h.

Loading fails LOUDLY: there is no CPU or PyTorch fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LIFT_LIB may point at an alternative build of the same ABI (A/B tuning runs only).
LIB_PATH = os.environ.get("LIFT_LIB") or os.path.join(_HERE, "liblift.so")

# Every symbol include/lift.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "lift_abi_version", "lift_status_string", "lift_workspace_bytes", "lift_scal",
    "lift_asum", "lift_dot", "lift_asum_partial", "lift_dot_partial", "lift_combine",
    "lift_gemv", "lift_debug_set_grid_limit", "lift_reduce_chunk_elems",
    "lift_reduce_group_chunks", "lift_blackscholes", "lift_scal_asum", "lift_xchg_bytes",
    "lift_xchg_create", "lift_xchg_destroy", "lift_ipc_get_handle", "lift_ipc_open_handle",
    "lift_ipc_close_handle", "lift_asum_allreduce", "lift_dot_allreduce", "lift_ipc_alloc",
    "lift_gemv_allgather", "lift_gemv_ws", "lift_gemv_workspace_bytes", "lift_set_variant",
    "lift_get_variant", "lift_last_cuda_error", "lift_workspace_check",
)

LIFT_OK = 0
ABI_VERSION = 1

_i64, _f32, _vp, _sz, _int = (ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.c_int)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"liblift.so not found at {LIB_PATH}: the CUDA extension is required (no CPU "
            "fallback). Build it with `python __graft_entry__.py`.")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "lift_abi_version": ([], _int),
        "lift_status_string": ([_int], ctypes.c_char_p),
        "lift_workspace_bytes": ([_i64], _sz),
        "lift_workspace_check": ([_vp, _sz, _vp], _int),
        "lift_scal": ([_i64, _f32, _vp, _vp, _vp], _int),
        "lift_asum": ([_i64, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_dot": ([_i64, _vp, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_asum_partial": ([_i64, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_dot_partial": ([_i64, _vp, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_combine": ([_int, _vp, _vp, _vp], _int),
        "lift_gemv": ([_i64, _i64, _f32, _vp, _i64, _vp, _f32, _vp, _vp, _vp], _int),
        "lift_gemv_ws": ([_i64, _i64, _f32, _vp, _i64, _vp, _f32, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_gemv_workspace_bytes": ([_i64, _i64], _sz),
        "lift_set_variant": ([_int, _int], _int),
        "lift_get_variant": ([_int], _int),
        "lift_last_cuda_error": ([], ctypes.c_char_p),
        "lift_debug_set_grid_limit": ([_int], _int),
        "lift_reduce_chunk_elems": ([], _i64),
        "lift_reduce_group_chunks": ([], _int),
        "lift_scal_asum": ([_i64, _f32, _vp, _vp, _vp, _vp, _sz, _vp], _int),
        "lift_xchg_bytes": ([_int], _sz),
        "lift_xchg_create": ([_int, ctypes.POINTER(ctypes.c_void_p)], _int),
        "lift_xchg_destroy": ([_vp], _int),
        "lift_ipc_get_handle": ([_vp, _vp], _int),
        "lift_ipc_open_handle": ([_vp, ctypes.POINTER(ctypes.c_void_p)], _int),
        "lift_ipc_close_handle": ([_vp], _int),
        "lift_asum_allreduce": ([_i64, _vp, _vp, _vp, _sz, _vp, _int, _int, ctypes.c_ulonglong,
                                 _vp, _vp], _int),
        "lift_dot_allreduce": ([_i64, _vp, _vp, _vp, _vp, _sz, _vp, _int, _int,
                                ctypes.c_ulonglong, _vp, _vp], _int),
        "lift_ipc_alloc": ([_sz, ctypes.POINTER(ctypes.c_void_p)], _int),
        "lift_gemv_allgather": ([_i64, _i64, _f32, _vp, _i64, _vp, _f32, _vp, _vp, _i64, _vp,
                                 _int, _int, ctypes.c_ulonglong, _vp, _vp], _int),
        "lift_blackscholes": ([_i64, _vp, _f32, _f32, _f32, _f32, _vp, _vp, _vp], _int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.lift_abi_version() != ABI_VERSION:
        raise ImportError(f"liblift.so ABI {L.lift_abi_version()} != {ABI_VERSION}")
    return L


lib = _load()


class LiftError(RuntimeError):
    pass


def check(status: int) -> None:
    if status != LIFT_OK:
        msg = lib.lift_status_string(status).decode()
        if status == 4:  # LIFT_ERR_CUDA: name the CUDA error behind it
            msg += f" ({lib.lift_last_cuda_error().decode()})"
        raise LiftError(msg)
