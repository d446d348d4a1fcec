"""paper_1502_02389_b200 — B200-native hot path of arXiv 1502.02389's BLAS compositions.

Thin Python binding over liblift.so (include/lift.h): argument marshalling only.
Every step of scal / asum / dot / gemv / combine runs in the sm_100a kernels behind
the C ABI; PyTorch supplies device memory, streams and (in ``dist``) process groups.

    scal(a, x)          = map(mult(a), x)
    asum(x)             = reduce(add, 0) o map(abs, x)
    dot(x, y)           = reduce(add, 0) o map(mult) o zip(x, y)
    gemv(A, x, y, a, b) = map(add) o zip(map(scal(a) o dot(x), A), scal(b, y))

Inputs must be fp32 CUDA tensors (vectors contiguous; A with unit column stride).
Violations raise ValueError; non-OK ABI statuses raise LiftError.  There is no CPU
fallback: a CPU tensor is an error, and a missing liblift.so fails at import.
"""
from __future__ import annotations

import contextlib
import os
import threading

import torch

from ._lib import LiftError, check, lib

__all__ = ["scal", "asum", "dot", "gemv", "asum_partial", "dot_partial", "combine", "blackscholes",
           "scal_asum",
           "workspace_bytes", "Workspace", "LiftError", "set_grid_limit", "set_variant",
           "get_variant", "VARIANTS"]


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_NULL_CTX = contextlib.nullcontext()


def _on(device: torch.device):
    """liblift launches on the CURRENT device (its SM count and occupancies too), so a call
    on another device's tensors runs with that device made current for its duration."""
    if device.index is None or device.index == torch.cuda.current_device():
        return _NULL_CTX
    return torch.cuda.device(device)


def _vec(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    if t.dim() != 1:
        raise ValueError(f"{name} must be 1-D")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


#: Debug aid for tests: allocate results pre-filled with NaN, so that an element a kernel
#: fails to write cannot pass by inheriting a correct value from a recycled allocation.
POISON_OUTPUTS = os.environ.get("LIFT_POISON_OUTPUTS", "") not in ("", "0")


def _out(out, n, dtype, device, name="out"):
    if out is None:
        if POISON_OUTPUTS:
            return torch.full((n,), float("nan"), dtype=dtype, device=device)
        return torch.empty(n, dtype=dtype, device=device)
    if (not out.is_cuda or out.dtype != dtype or out.numel() != n or not out.is_contiguous()
            or out.device != device):
        raise ValueError(f"{name} must be a contiguous {dtype} CUDA tensor of {n} elements")
    return out


#: canonical reduction decomposition (lift_reduce_chunk_elems / _group_chunks)
CHUNK_ELEMS = int(lib.lift_reduce_chunk_elems())
GROUP_CHUNKS = int(lib.lift_reduce_group_chunks())
GROUP_ELEMS = CHUNK_ELEMS * GROUP_CHUNKS


def workspace_bytes(n: int) -> int:
    return int(lib.lift_workspace_bytes(int(n)))


class Workspace:
    """Zero-filled reduction workspace (the caller-owned buffer of lift.h).

    Zero-filled once at allocation; every lift call leaves its tickets at zero, so
    it is reusable.  Use one per stream.
    """

    def __init__(self, n: int, device):
        self.nbytes = workspace_bytes(n)
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def reset(self) -> None:
        """Zero-fill again (clears the tickets)."""
        self.buf.zero_()

    def check(self) -> bool:
        """lift_workspace_check: True if every last-block-done ticket is zero (the contract
        holds); False if a call was aborted or overlapped on this buffer (then reset()).
        Synchronises with the current stream; off the hot path."""
        dev = self.buf.device
        with _on(dev):
            st = lib.lift_workspace_check(self.ptr, self.nbytes, _stream_handle(dev))
        if st == 3:  # LIFT_ERR_WORKSPACE
            return False
        check(st)
        return True


_ws_lock = threading.Lock()
_ws_cache: dict = {}


def _workspace(n: int, device: torch.device) -> Workspace:
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    need = workspace_bytes(n)
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.nbytes < need:
            ws = Workspace(n, device)
            _ws_cache[key] = ws
        return ws


def set_grid_limit(max_ctas: int) -> None:
    """Test hook (lift_debug_set_grid_limit): cap CTAs per launch; 0 = no cap."""
    check(lib.lift_debug_set_grid_limit(int(max_ctas)))


#: NEXT-4 runtime strategy knobs (lift.h lift_variant); every value gives the same bits.
VARIANTS = {"load_width": 0, "gemv_x": 1, "prefetch": 2, "order": 3, "stagger": 4}


def set_variant(knob: str, value: int) -> None:
    """Select a strategy variant (lift_set_variant); 0 restores the tuned default."""
    check(lib.lift_set_variant(VARIANTS[knob], int(value)))


def get_variant(knob: str) -> int:
    return int(lib.lift_get_variant(VARIANTS[knob]))


def scal(alpha: float, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """y = alpha * x (lift_scal).  ``out`` may be ``x`` itself (in place)."""
    x = _vec(x, "x")
    y = _out(out, x.numel(), torch.float32, x.device)
    with _on(x.device):
        check(lib.lift_scal(x.numel(), float(alpha), x.data_ptr(), y.data_ptr(),
                            _stream_handle(x.device)))
    return y


def asum(x: torch.Tensor, out: torch.Tensor | None = None,
         ws: Workspace | None = None) -> torch.Tensor:
    """1-element fp32 tensor = sum |x_i| (lift_asum)."""
    x = _vec(x, "x")
    r = _out(out, 1, torch.float32, x.device)
    w = ws or _workspace(x.numel(), x.device)
    with _on(x.device):
        check(lib.lift_asum(x.numel(), x.data_ptr(), r.data_ptr(), w.ptr, w.nbytes,
                            _stream_handle(x.device)))
    return r


def dot(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None,
        ws: Workspace | None = None) -> torch.Tensor:
    """1-element fp32 tensor = sum x_i*y_i (lift_dot).  zip needs equal lengths."""
    x, y = _vec(x, "x"), _vec(y, "y")
    if x.numel() != y.numel():
        raise ValueError("zip-length-mismatch: dot needs equal lengths (PAPER.md P:307)")
    if x.device != y.device:
        raise ValueError("x and y must be on the same device")
    r = _out(out, 1, torch.float32, x.device)
    w = ws or _workspace(x.numel(), x.device)
    with _on(x.device):
        check(lib.lift_dot(x.numel(), x.data_ptr(), y.data_ptr(), r.data_ptr(), w.ptr, w.nbytes,
                           _stream_handle(x.device)))
    return r


def scal_asum(alpha: float, x: torch.Tensor, out: torch.Tensor | None = None,
              result: torch.Tensor | None = None, ws: Workspace | None = None):
    """Fused y = alpha*x and asum(y) in one pass (lift_scal_asum).  Returns (y, result);
    bit-identical to (scal(alpha, x), asum(scal(alpha, x))).  ``out`` must not be ``x``."""
    x = _vec(x, "x")
    y = _out(out, x.numel(), torch.float32, x.device)
    r = _out(result, 1, torch.float32, x.device, "result")
    w = ws or _workspace(x.numel(), x.device)
    with _on(x.device):
        check(lib.lift_scal_asum(x.numel(), float(alpha), x.data_ptr(), y.data_ptr(), r.data_ptr(),
                                 w.ptr, w.nbytes, _stream_handle(x.device)))
    return y, r


def asum_partial(x: torch.Tensor, out: torch.Tensor | None = None,
                 ws: Workspace | None = None) -> torch.Tensor:
    """1-element fp64 tensor: the un-rounded asum total (lift_asum_partial)."""
    x = _vec(x, "x")
    r = _out(out, 1, torch.float64, x.device)
    w = ws or _workspace(x.numel(), x.device)
    with _on(x.device):
        check(lib.lift_asum_partial(x.numel(), x.data_ptr(), r.data_ptr(), w.ptr, w.nbytes,
                                    _stream_handle(x.device)))
    return r


def dot_partial(x: torch.Tensor, y: torch.Tensor, out: torch.Tensor | None = None,
                ws: Workspace | None = None) -> torch.Tensor:
    """1-element fp64 tensor: the un-rounded dot total (lift_dot_partial)."""
    x, y = _vec(x, "x"), _vec(y, "y")
    if x.numel() != y.numel():
        raise ValueError("zip-length-mismatch: dot needs equal lengths (PAPER.md P:307)")
    r = _out(out, 1, torch.float64, x.device)
    w = ws or _workspace(x.numel(), x.device)
    with _on(x.device):
        check(lib.lift_dot_partial(x.numel(), x.data_ptr(), y.data_ptr(), r.data_ptr(), w.ptr,
                                   w.nbytes, _stream_handle(x.device)))
    return r


def combine(partials: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """1-element fp32 tensor = RN(pairwise sum of fp64 partials) (lift_combine)."""
    if not (isinstance(partials, torch.Tensor) and partials.is_cuda
            and partials.dtype == torch.float64 and partials.is_contiguous()
            and partials.numel() >= 1):
        raise ValueError("partials must be a non-empty contiguous float64 CUDA tensor")
    r = _out(out, 1, torch.float32, partials.device)
    with _on(partials.device):
        check(lib.lift_combine(partials.numel(), partials.data_ptr(), r.data_ptr(),
                               _stream_handle(partials.device)))
    return r


def gemv(A: torch.Tensor, x: torch.Tensor, y: torch.Tensor, alpha: float, beta: float,
         out: torch.Tensor | None = None, split: bool = True) -> torch.Tensor:
    """y_out = alpha * A @ x + beta * y (lift_gemv_ws), A row-major (stride(1) == 1).

    ``out`` may be ``y`` (in place).  ``split=False`` withholds the workspace, forcing one
    CTA per row for long rows (same bits; for tests)."""
    if not (isinstance(A, torch.Tensor) and A.is_cuda and A.dtype == torch.float32
            and A.dim() == 2):
        raise ValueError("A must be a 2-D float32 CUDA tensor")
    m, n = A.shape
    if m > 0 and n > 0 and A.stride(1) != 1:
        raise ValueError("A must be row-major with unit column stride")
    lda = A.stride(0) if (m > 1 and n > 0) else max(1, n)
    x, y = _vec(x, "x"), _vec(y, "y")
    if x.numel() != n or y.numel() != m:
        raise ValueError(f"dimension-mismatch: A is {m}x{n}, x has {x.numel()}, "
                         f"y has {y.numel()}")
    yo = _out(out, m, torch.float32, A.device)
    with _on(A.device):
        need = int(lib.lift_gemv_workspace_bytes(m, n)) if split else 0  # device's SM count
        wp, wb = (0, 0)
        if need:  # rows >= 65536 columns: the split path needs a workspace (lift_gemv_ws)
            w = _gemv_workspace(need, A.device)
            wp, wb = w.data_ptr(), w.numel()
        check(lib.lift_gemv_ws(m, n, float(alpha), A.data_ptr(), lda, x.data_ptr(), float(beta),
                               y.data_ptr(), yo.data_ptr(), wp or None, wb,
                               _stream_handle(A.device)))
    return yo


_gemv_ws_cache: dict = {}


def _gemv_workspace(need: int, device: torch.device) -> torch.Tensor:
    """Zero-filled gemv split-path workspace per (device, stream), grown on demand."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    with _ws_lock:
        w = _gemv_ws_cache.get(key)
        if w is None or w.numel() < need:
            w = torch.zeros(need, dtype=torch.uint8, device=device)
            _gemv_ws_cache[key] = w
        return w


def blackscholes(s: torch.Tensor, K: float, r: float, v: float, T: float,
                 call: torch.Tensor | None = None, put: torch.Tensor | None = None):
    """(call, put) = map(BSComputation, s) (lift_blackscholes; Fig. 9)."""
    s = _vec(s, "s")
    c = _out(call, s.numel(), torch.float32, s.device, "call")
    p = _out(put, s.numel(), torch.float32, s.device, "put")
    with _on(s.device):
        check(lib.lift_blackscholes(s.numel(), s.data_ptr(), float(K), float(r), float(v), float(T),
                                    c.data_ptr(), p.data_ptr(), _stream_handle(s.device)))
    return c, p
