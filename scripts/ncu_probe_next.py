"""ncu driver for the NEXT-row kernels: fused scal+asum (2^28) and BlackScholes (4M)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
x = gen.fill_device(torch.empty(1 << 28, device=dev), 0, 1, 0, 0, -1.0, 1.0)
y = torch.empty_like(x)
s = gen.fill_device(torch.empty(4 << 20, device=dev), 0, 1, 0, 0, 10.0, 200.0)
r = torch.empty(1, device=dev)
ws = lift.Workspace(1 << 28, dev)
for _ in range(2):
    lift.scal_asum(3.0, x, out=y, result=r, ws=ws)
    lift.blackscholes(s, 100.0, 0.05, 0.2, 1.0)
torch.cuda.synchronize()
