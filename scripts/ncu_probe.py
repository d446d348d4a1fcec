"""Small driver for ncu: each op of the bench step at bench size, a few launches each
(inputs device-generated).  Usage: ncu ... python scripts/ncu_probe.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda:0")


def fill(n, tid, lo, hi):
    return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, 0, 0, lo, hi)


x = fill(1 << 28, 1, -1.0, 1.0)
y = torch.empty(1 << 28, dtype=torch.float32, device=dev)
dx = fill(1 << 26, 1, 0.0, 1.0)
dy = fill(1 << 26, 2, 0.0, 2.0)
A = fill(8192 * 8192, 3, 0.0, 3.0).view(8192, 8192)
gx = fill(8192, 1, 0.0, 1.0)
gy = fill(8192, 2, 0.0, 2.0)
go = torch.empty(8192, dtype=torch.float32, device=dev)
r = torch.empty(1, dtype=torch.float32, device=dev)
ws = lift.Workspace(1 << 28, dev)
torch.cuda.synchronize()
for _ in range(reps):
    lift.scal(3.0, x, out=y)
    lift.asum(x, out=r, ws=ws)
    lift.dot(dx, dy, out=r, ws=ws)
    lift.gemv(A, gx, gy, 1.5, 0.5, out=go)
torch.cuda.synchronize()
print("probe done", r.item())
