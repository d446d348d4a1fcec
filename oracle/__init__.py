"""CPU oracle (fp64, Neumaier) for scal / asum / dot / gemv — see oracle.c.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product package ``paper_1502_02389_b200`` never does, and the
two share no code (only the seeded generator in ``lift_inputs`` feeds both).

Every function follows the paper's plain definition;
each C function cites its line.  Results are returned in fp64; callers round
to fp32 once (``np.float32(v)``) for the bit-exact comparisons.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_scal.argtypes = [ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_scal.restype = None
        L.oracle_asum.argtypes = [ctypes.c_int64, ctypes.c_void_p]
        L.oracle_asum.restype = ctypes.c_double
        L.oracle_asum_acc.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_asum_acc.restype = None
        L.oracle_dot.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_dot.restype = ctypes.c_double
        L.oracle_dot_acc.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p]
        L.oracle_dot_acc.restype = None
        L.oracle_gemv.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_float,
                                  ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                  ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_gemv.restype = None
        L.oracle_blackscholes.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_blackscholes.restype = None
        L.oracle_finish.argtypes = [ctypes.c_void_p]
        L.oracle_finish.restype = ctypes.c_double
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def scal(alpha: float, x) -> np.ndarray:
    """returns fp64 alpha*x_i (exact)."""
    x = _f32(x)
    y = np.empty(x.size, np.float64)
    lib().oracle_scal(x.size, np.float32(alpha), x.ctypes.data, y.ctypes.data)
    return y


def asum(x) -> float:
    """fp64 compensated sum of abs(x_i)."""
    x = _f32(x)
    return lib().oracle_asum(x.size, x.ctypes.data)


def dot(x, y) -> float:
    """fp64 compensated sum of x_i*y_i (zip needs equal lengths)."""
    x, y = _f32(x), _f32(y)
    if x.size != y.size:
        raise ValueError("zip-length-mismatch: dot needs equal lengths (P:307)")
    return lib().oracle_dot(x.size, x.ctypes.data, y.ctypes.data)


class Stream:
    """Streaming asum/dot over blocks (for sizes too large to hold on the host).

    Same left fold as ``asum``/``dot``; the Neumaier state (s, c) carries over
    between blocks, so the result equals the one-shot call on the concatenation.
    """

    def __init__(self):
        self.state = np.zeros(2, np.float64)

    def asum(self, x):
        x = _f32(x)
        lib().oracle_asum_acc(x.size, x.ctypes.data, self.state.ctypes.data)

    def dot(self, x, y):
        x, y = _f32(x), _f32(y)
        assert x.size == y.size
        lib().oracle_dot_acc(x.size, x.ctypes.data, y.ctypes.data, self.state.ctypes.data)

    def value(self) -> float:
        return float(lib().oracle_finish(self.state.ctypes.data))


def gemv(A, x, y, alpha: float, beta: float) -> np.ndarray:
    """P:796-798 / P:814 — out = alpha*A@x + beta*y, A row-major (reading R8)."""
    A = np.asarray(A, dtype=np.float32)
    if A.ndim != 2:
        raise ValueError("A must be 2-D")
    m, n = A.shape
    if A.strides[1] != 4 or A.strides[0] % 4:
        A = np.ascontiguousarray(A)
    lda = A.strides[0] // 4 if m > 0 else n
    x, y = _f32(x), _f32(y)
    if x.size != n or y.size != m:
        raise ValueError("dimension-mismatch")
    out = np.empty(m, np.float64)
    lib().oracle_gemv(m, n, np.float32(alpha), A.ctypes.data, lda, x.ctypes.data,
                      np.float32(beta), y.ctypes.data, out.ctypes.data)
    return out


def blackscholes(s, K: float, r: float, v: float, T: float):
    """Fig. 9 map(BSComputation, s): fp64 (call, put) per stock price."""
    s = _f32(s)
    call = np.empty(s.size, np.float64)
    put = np.empty(s.size, np.float64)
    lib().oracle_blackscholes(s.size, s.ctypes.data, float(K), float(r), float(v), float(T),
                              call.ctypes.data, put.ctypes.data)
    return call, put
