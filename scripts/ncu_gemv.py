"""One gemv launch at m x n for an ncu capture: python scripts/ncu_gemv.py [m] [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device("cuda:0")
A = gen.fill_device(torch.empty(m * n, device=dev), 0, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
x = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
y = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
o = torch.empty(m, device=dev)
if os.environ.get("LIFT_PF"):  # LIFT_VAR_PREFETCH: 1 off, 2 on
    lift.set_variant("prefetch", int(os.environ["LIFT_PF"]))
if os.environ.get("GEMV_X"):  # LIFT_VAR_GEMV_X: 1 = x via L1, 2 = x staged fp64 in smem
    lift.set_variant("gemv_x", int(os.environ["GEMV_X"]))
for _ in range(3):
    lift.gemv(A, x, y, 1.5, 0.5, out=o)
torch.cuda.synchronize()
print("ok")
