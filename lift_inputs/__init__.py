"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no scal/asum/dot/gemv).  It
only turns ``(seed, tensor id, global element index)`` into an fp32 value, so
that the oracle (``oracle/``) and the CUDA path (``paper_1502_02389_b200``)
can be fed bit-identical inputs without either importing the other.

Recipe:

    z   = seed*0x9E3779B97F4A7C15 + tid*0xD1B54A32D192ED03 + i     (mod 2^64)
    raw = splitmix64_mix(z + 0x9E3779B97F4A7C15)                    (Vigna's finaliser)
    uniform(lo, hi):  u = (raw >> 40) * 2^-24          (exact, 24 bits, [0, 1))
                      v = fp32_RN( lo + (hi - lo) * u ) (two fp64 RN ops, no FMA)
    integer:          v = fp32( ((raw >> 32) mod 17) - 8 )  in {-8 .. 8}

``i`` is the GLOBAL element index, so a shard ``[i0, i0+n)`` generated on any
rank is the same slice of the same global vector (sharding-independent).
For a row-major matrix with ``lda == ncols`` element ``(r, c)`` has
``i = r*ncols + c``.

Three implementations of the same recipe exist:
  * ``*_np``    — numpy, the readable specification (used for small sizes and
                  to pin the other two);
  * host C      — ``gen_host.c`` → ``liblift_inputs_host.so`` (fast, for the
                  oracle at large sizes);
  * device CUDA — ``gen_device.cu`` → ``liblift_inputs_dev.so`` (fills device
                  buffers for the GPU tests and bench).
Tests assert all three agree bit for bit.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
ID_MUL = 0xD1B54A32D192ED03
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

# tensor ids
TID_X, TID_Y, TID_A = 1, 2, 3

# distribution codes shared with the C / CUDA twins
DIST_UNIFORM = 0
DIST_INT17 = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "liblift_inputs_host.so")
DEV_LIB = os.path.join(_HERE, "liblift_inputs_dev.so")


# ---------------------------------------------------------------- numpy spec
def raw_np(seed: int, tid: int, i0: int, n: int) -> np.ndarray:
    """64-bit counter-based draws for global indices i0 .. i0+n-1 (numpy spec)."""
    with np.errstate(over="ignore"):
        base = np.uint64((seed * GOLDEN + tid * ID_MUL + i0) & 0xFFFFFFFFFFFFFFFF)
        z = base + np.arange(n, dtype=np.uint64)
        z = z + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_np(seed: int, tid: int, i0: int, n: int, lo: float, hi: float) -> np.ndarray:
    u = (raw_np(seed, tid, i0, n) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)
    v = np.float64(lo) + np.float64(hi - lo) * u  # numpy never contracts to FMA
    return v.astype(np.float32)


def int17_np(seed: int, tid: int, i0: int, n: int) -> np.ndarray:
    r = (raw_np(seed, tid, i0, n) >> np.uint64(32)) % np.uint64(17)
    return (r.astype(np.int64) - 8).astype(np.float32)


# ------------------------------------------------------------------ host C twin
_host = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(HOST_LIB)
        lib.lift_inputs_fill_host.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
            ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_double]
        lib.lift_inputs_fill_host.restype = ctypes.c_int
        _host = lib
    return _host


def fill_host(out: np.ndarray, seed: int, tid: int, i0: int, dist: int = DIST_UNIFORM,
              lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Fill a contiguous fp32 numpy array in place with global indices i0.."""
    assert out.dtype == np.float32 and out.flags.c_contiguous
    rc = _host_lib().lift_inputs_fill_host(out.ctypes.data, out.size, seed, tid, i0,
                                           dist, lo, hi)
    if rc != 0:
        raise RuntimeError(f"lift_inputs_fill_host failed ({rc})")
    return out


def host(n: int, seed: int, tid: int, i0: int = 0, dist: int = DIST_UNIFORM,
         lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return fill_host(np.empty(n, np.float32), seed, tid, i0, dist, lo, hi)


# --------------------------------------------------------------- device twin
_dev = None


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError(f"{DEV_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(DEV_LIB)
        lib.lift_inputs_fill_device.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
            ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        lib.lift_inputs_fill_device.restype = ctypes.c_int
        _dev = lib
    return _dev


def fill_device(t, seed: int, tid: int, i0: int = 0, dist: int = DIST_UNIFORM,
                lo: float = -1.0, hi: float = 1.0):
    """Fill a contiguous fp32 CUDA torch tensor in place (on its current stream)."""
    import torch
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    stream = torch.cuda.current_stream(t.device).cuda_stream
    rc = _dev_lib().lift_inputs_fill_device(t.data_ptr(), t.numel(), seed, tid, i0,
                                            dist, lo, hi, stream)
    if rc != 0:
        raise RuntimeError(f"lift_inputs_fill_device failed ({rc})")
    return t
