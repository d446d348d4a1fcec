"""X1 — sharding across GPUs (one process per GPU, torch.distributed over NCCL).

The paper runs on one device; sharding comes from BASELINE.json's
north star: "Each rank reduces its shard, and one NCCL allreduce of a scalar, or a
gather of y slices over NVLink, combines them."

  scal  — contiguous shards, independent: NO collective.
  asum, dot — each rank folds its shard to an fp64 partial (lift_*_partial); ONE
          exchange (all-gather of p x 8 bytes) and a fixed-order pairwise combine
          (lift_combine) give every rank the same fp32 bits.  We gather instead of
          all-reducing so the combine order never depends on NCCL's algorithm
          (ring / tree / NVLS); the cost is identical at 8 bytes per rank.
  gemv  — rows are sharded, x is replicated (each rank generates or holds it), y is
          sharded; ONE exchange: all-gather of the y_out slices.

Shard boundaries for reductions are aligned to the canonical group size
(RED_G * RED_C = 2^21 elements) when possible, so that with a power-of-two number of
groups per rank the combined result is bit-identical to the unsharded one
(reading R5).

The collective plumbing is kept separate from the CUDA calls (``gather_partials``,
``gather_rows``) so it can be exercised with the gloo backend on CPU; the combine
itself always runs in liblift (``combine_fn`` is injectable only for those tests).
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import GROUP_ELEMS  # noqa: E402  (RED_G * RED_C from liblift, csrc/canon.h)


def shard_range(n: int, rank: int, world: int, align: int = GROUP_ELEMS) -> tuple[int, int]:
    """Contiguous [start, stop) of rank `rank` in a length-n vector.

    Boundaries are multiples of `align` (the last rank takes the remainder) when n is
    large enough that every rank gets at least one aligned block; otherwise an even
    split.  The ranges tile [0, n) exactly, in rank order."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard request")
    if align > 1 and n >= align * world:
        blocks = -(-n // align)
        per = blocks // world
        extra = blocks % world
        b0 = rank * per + min(rank, extra)
        b1 = b0 + per + (1 if rank < extra else 0)
        return min(n, b0 * align), min(n, b1 * align)
    base, rem = divmod(n, world)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


def row_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [start, stop) owned by `rank` for gemv (even split, rank order)."""
    return shard_range(m, rank, world, align=1)


def _world(group):
    return dist.get_world_size(group) if dist.is_initialized() else 1


def gather_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather one fp64 partial per rank into a rank-ordered [p] tensor."""
    p = _world(group)
    if not dist.is_initialized():
        return partial.reshape(1)
    out = torch.empty(p, dtype=partial.dtype, device=partial.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, partial.reshape(1), group=group)
    else:
        parts = [torch.empty(1, dtype=partial.dtype, device=partial.device) for _ in range(p)]
        dist.all_gather(parts, partial.reshape(1), group=group)
        out.copy_(torch.cat(parts))
    return out


def gather_rows(y_slice: torch.Tensor, m: int, group=None, out: torch.Tensor | None = None):
    """All-gather rank-ordered y slices (row_range split) into the full length-m y."""
    p = _world(group)
    if out is None:
        out = torch.empty(m, dtype=y_slice.dtype, device=y_slice.device)
    if not dist.is_initialized():
        out.copy_(y_slice)
        return out
    rank = dist.get_rank(group)
    sizes = [row_range(m, r, p)[1] - row_range(m, r, p)[0] for r in range(p)]
    if y_slice.numel() != sizes[rank]:
        raise ValueError("y slice does not match row_range")
    if len(set(sizes)) == 1 and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, y_slice, group=group)
        return out
    mx = max(sizes)
    padded = torch.zeros(mx, dtype=y_slice.dtype, device=y_slice.device)
    padded[:y_slice.numel()] = y_slice
    parts = [torch.empty(mx, dtype=y_slice.dtype, device=y_slice.device) for _ in range(p)]
    dist.all_gather(parts, padded, group=group)
    out.copy_(torch.cat([parts[r][:sizes[r]] for r in range(p)]))
    return out


def _lift():
    import paper_1502_02389_b200 as lift
    return lift


def sharded_scal(alpha: float, x_shard: torch.Tensor, out=None):
    """scal needs no exchange: each rank scales its own shard."""
    return _lift().scal(alpha, x_shard, out=out)


def sharded_asum(x_shard: torch.Tensor, group=None, combine_fn=None, out=None, ws=None):
    lift = _lift()
    part = lift.asum_partial(x_shard, ws=ws)
    allp = gather_partials(part, group)
    return (combine_fn or lift.combine)(allp, out=out)


def sharded_dot(x_shard: torch.Tensor, y_shard: torch.Tensor, group=None, combine_fn=None,
                out=None, ws=None):
    lift = _lift()
    part = lift.dot_partial(x_shard, y_shard, ws=ws)
    allp = gather_partials(part, group)
    return (combine_fn or lift.combine)(allp, out=out)


def sharded_gemv(A_rows: torch.Tensor, x: torch.Tensor, y_rows: torch.Tensor, alpha: float,
                 beta: float, m: int, group=None, out_full=None, out_slice=None):
    """Each rank computes its rows' y_out slice, then all ranks gather the full y."""
    ys = _lift().gemv(A_rows, x, y_rows, alpha, beta, out=out_slice)
    return gather_rows(ys, m, group, out=out_full)


class PeerExchange:
    """NEXT-1: the cross-GPU combine fused into the reduction kernel (lift_*_allreduce).

    Each rank creates an exchange buffer (lift_xchg_create), exports it with CUDA IPC,
    and maps every peer's buffer; the reduction's final CTA then writes its fp64 partial
    straight into the peers' buffers (NVLink P2P stores on a multi-GPU node), waits for
    theirs and folds them in rank order — no separate NCCL launch, same bits on every
    rank as ``sharded_asum``/``sharded_dot``.  The 64-byte IPC handles are exchanged
    once, through ``torch.distributed`` (any backend).  All ranks must call ``asum`` /
    ``dot`` in the same sequence.
    """

    def __init__(self, group=None, device=None):
        from ._lib import check, lib
        self._lib, self._check = lib, check
        self.group = group
        self.p = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        buf = ctypes.c_void_p()
        check(lib.lift_xchg_create(self.p, ctypes.byref(buf)))
        self.buf = buf.value
        ptrs, self.opened = self._share(self.buf)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        self.error = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.epoch = 0
        self._y = None  # (m, own ptr, opened peer ptrs, device array, tensor view)

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def asum(self, x_shard, out=None, ws=None):
        lift = _lift()
        x = lift._vec(x_shard, "x")
        r = lift._out(out, 1, torch.float32, x.device)
        w = ws or lift._workspace(x.numel(), x.device)
        self.epoch += 1  # the ABI needs epoch = previous + 1 per exchange buffer (bank parity)
        with torch.cuda.device(self.device):
            self._check(self._lib.lift_asum_allreduce(
                x.numel(), x.data_ptr(), r.data_ptr(), w.ptr, w.nbytes, self.peers.data_ptr(),
                self.p, self.rank, self.epoch, self.error.data_ptr(), self._stream()))
        return r

    def dot(self, x_shard, y_shard, out=None, ws=None):
        lift = _lift()
        x, y = lift._vec(x_shard, "x"), lift._vec(y_shard, "y")
        if x.numel() != y.numel():
            raise ValueError("zip-length-mismatch: dot needs equal lengths (PAPER.md P:307)")
        r = lift._out(out, 1, torch.float32, x.device)
        w = ws or lift._workspace(x.numel(), x.device)
        self.epoch += 1
        with torch.cuda.device(self.device):
            self._check(self._lib.lift_dot_allreduce(
                x.numel(), x.data_ptr(), y.data_ptr(), r.data_ptr(), w.ptr, w.nbytes,
                self.peers.data_ptr(), self.p, self.rank, self.epoch, self.error.data_ptr(),
                self._stream()))
        return r

    def _share(self, own_ptr):
        """Exchange IPC handles of `own_ptr` (a lift-allocated base pointer); returns
        the p pointers (own at `rank`) and the list of opened peer mappings."""
        handle = (ctypes.c_ubyte * 64)()
        self._check(self._lib.lift_ipc_get_handle(own_ptr, handle))
        handles = [bytes(handle)]
        if self.p > 1:
            handles = [None] * self.p
            dist.all_gather_object(handles, bytes(handle), group=self.group)
        ptrs, opened = [], []
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs.append(own_ptr)
                continue
            ptr = ctypes.c_void_p()
            self._check(self._lib.lift_ipc_open_handle(
                (ctypes.c_ubyte * 64).from_buffer_copy(h), ctypes.byref(ptr)))
            opened.append(ptr.value)
            ptrs.append(ptr.value)
        return ptrs, opened

    def _full_y(self, m: int):
        """Two banks (epoch parity) of a full-length y per rank, IPC-shared: a peer can be at
        most one call ahead (finishing call e needs every rank's call-e rows), so it writes
        call e+1's rows into the other bank while this rank may still read call e's."""
        if self._y is not None and self._y[0] == m:
            return self._y
        self._free_y()
        buf = ctypes.c_void_p()
        self._check(self._lib.lift_ipc_alloc(max(8, 8 * m), ctypes.byref(buf)))
        ptrs, opened = self._share(buf.value)
        arrs = [torch.tensor([p + 4 * m * b for p in ptrs], dtype=torch.int64, device=self.device)
                for b in (0, 1)]
        base = torch.as_tensor(_DevArray(buf.value, 2 * m, self.device.index), device=self.device)
        views = [base[:m], base[m:]]
        self._y = (m, buf.value, opened, arrs, views)
        return self._y

    def _free_y(self):
        if self._y is None:
            return
        torch.cuda.synchronize(self.device)
        if self.p > 1 and dist.is_initialized():
            dist.barrier(group=self.group)
        for ptr in self._y[2]:
            self._lib.lift_ipc_close_handle(ptr)
        self._lib.lift_xchg_destroy(self._y[1])
        self._y = None

    def gemv(self, A_rows, x, y_rows, alpha: float, beta: float, m: int, row0: int):
        """y_full = alpha*A@x + beta*y over all ranks' rows, the all-gather fused into the
        gemv kernel (lift_gemv_allgather).  Returns this rank's full-length y: a view of
        the IPC-shared bank of this call (banks alternate by call).  It stays valid until
        this rank's next-but-one call; work enqueued on this stream before the next call
        may read it.  Every rank must own >= 1 row (m >= world)."""
        lift = _lift()
        if not (A_rows.is_cuda and A_rows.dtype == torch.float32 and A_rows.dim() == 2):
            raise ValueError("A must be a 2-D float32 CUDA tensor")
        ml, n = A_rows.shape
        if ml > 0 and n > 0 and A_rows.stride(1) != 1:
            raise ValueError("A must be row-major with unit column stride")
        if m < self.p:
            raise ValueError(f"fused all-gather needs m >= world ({m} < {self.p}): every rank "
                             "must own at least one row")
        lda = A_rows.stride(0) if (ml > 1 and n > 0) else max(1, n)
        x, y = lift._vec(x, "x"), lift._vec(y_rows, "y")
        if x.numel() != n or y.numel() != ml:
            raise ValueError("dimension-mismatch")
        if ml == 0:
            raise ValueError("this rank owns no rows (use row_range)")
        _, _, _, arrs, views = self._full_y(m)
        self.epoch += 1
        bank = self.epoch & 1
        with torch.cuda.device(self.device):
            self._check(self._lib.lift_gemv_allgather(
                ml, n, float(alpha), A_rows.data_ptr(), lda, x.data_ptr(), float(beta),
                y.data_ptr(), arrs[bank].data_ptr(), row0, self.peers.data_ptr(), self.p,
                self.rank, self.epoch, self.error.data_ptr(), self._stream()))
        return views[bank]

    def check(self):
        """Raise if any exchange of this object timed out (a peer missed an epoch): the
        kernel then returned NaN (asum/dot) or an incomplete y (gemv) and set the error
        word.  Synchronises this device."""
        if int(self.error.item()) != 0:
            raise RuntimeError("PeerExchange: a peer did not arrive within the bounded wait "
                               "(~10 s); results of the affected calls are invalid")

    def close(self):
        self._free_y()
        torch.cuda.synchronize(self.device)
        err = int(self.error.item()) if self.error is not None else 0
        if self.p > 1 and dist.is_initialized():
            dist.barrier(group=self.group)  # nobody still writes into our buffer
        for ptr in self.opened:
            self._lib.lift_ipc_close_handle(ptr)
        self.opened = []
        if self.buf:
            self._lib.lift_xchg_destroy(self.buf)
            self.buf = None
        if err:
            raise RuntimeError("PeerExchange: a peer exchange timed out during this object's "
                               "lifetime; see check()")


class _DevArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view a lift-allocated buffer."""

    def __init__(self, ptr: int, n: int, device_index: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}
        self.device_index = device_index
