"""Small invocations of every kernel and launch path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):  compute-sanitizer --tool <t> python scripts/sanitize_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device="cpu").manual_seed(0)


def rnd(n, off=0):
    buf = torch.empty(n + off + 8, device=dev)
    v = buf[off:off + n]
    v.copy_(torch.rand(n, generator=g) * 2 - 1)
    return v


C = lift.CHUNK_ELEMS
for n, off in [(0, 0), (1, 0), (13, 3), (C + 5, 0), (C + 5, 1), (2 * lift.GROUP_ELEMS + 77, 4)]:
    x, y = rnd(n, off), rnd(n, (off * 3) % 8)
    lift.scal(3.0, x)
    lift.scal(3.0, x, out=x)
    lift.asum(x), lift.dot(x, y), lift.asum_partial(x), lift.dot_partial(x, y)
    if n:
        out = torch.empty(n + 8, device=dev)[1:1 + n] if off else None
        lift.scal_asum(2.0, x, out=out)
        lift.blackscholes(x.abs() + 1.0, 1.5, 0.05, 0.2, 1.0)
lift.combine(torch.rand(5, dtype=torch.float64, device=dev))
x = rnd(1000)
x[7] = float("inf")
lift.asum(x)  # fp64 refold path
for m, n, pad in [(3, 5, 0), (40, 1000, 3), (30, 3001, 1), (9, 4100, 0), (40, 8192, 0), (6, 8195, 2),
                 (17, 9000, 4), (5, 20000, 0)]:
    A = torch.rand(m, n + pad, generator=g).to(dev)[:, :n]
    lift.gemv(A, rnd(n), rnd(m), 1.5, 0.5)
# long rows: split path (few rows, workspace) twice (ticket reset), one CTA per row
for m, n, split in [(2, 65536 + 5, True), (1, 1 << 19, True), (2, 65536 + 5, True),
                    (3, 70001, False), (600, 65536, True)]:
    A = torch.rand(m, n, generator=g).to(dev)
    lift.gemv(A, rnd(n), rnd(m), 1.5, 0.5, split=split)
# round-2 kernels: staged-x gemv (register ring, TMA ring), prefetch on/off, 128-bit loads
for var in (2, 3):
    lift.set_variant("gemv_x", var)
    for m, n in [(37, 2048), (9, 4096), (70, 8192), (3, 16384)]:
        A = torch.rand(m, n, generator=g).to(dev)
        lift.gemv(A, rnd(n), rnd(m), 1.5, 0.5)
lift.set_variant("gemv_x", 0)
for pf in (1, 2):
    lift.set_variant("prefetch", pf)
    x = rnd(3 * C + 11)
    lift.scal(3.0, x), lift.asum(x), lift.scal_asum(2.0, x)
    A = torch.rand(1100, 4096, generator=g).to(dev)
    lift.gemv(A, rnd(4096), rnd(1100), 1.5, 0.5)
lift.set_variant("prefetch", 0)
lift.set_variant("load_width", 4)
x, y = rnd(C + 77), rnd(C + 77)
lift.scal(3.0, x), lift.dot(x, y)
lift.set_variant("load_width", 0)
# launches with more units than resident CTAs: the first-wave stagger (default on for the
# reductions and the x-in-shared-memory gemv; 4 = also scal and the x-through-L1 gemv)
for st in (0, 4):
    lift.set_variant("stagger", st)
    x, y = rnd((1 << 23) + 13), rnd((1 << 23) + 13)
    lift.asum(x), lift.dot(x, y), lift.scal(3.0, x), lift.scal_asum(2.0, x)
    A = torch.rand(4100, 2048, generator=g).to(dev)
    lift.gemv(A, rnd(2048), rnd(4100), 1.5, 0.5)
lift.set_variant("stagger", 0)
torch.cuda.synchronize()
print("sanitize probe ok")
