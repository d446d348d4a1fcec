"""Interleaved A/B of a runtime knob on the bench step (scal 2^28, asum 2^28, dot 2^26,
gemv 8192^2, no events between kernels): python scripts/step_knob_ab.py knob v1,v2,... [K]
Each repetition times K back-to-back steps per knob value, values interleaved, 9 reps;
prints the median ms/step and GB/s per value."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

knob = sys.argv[1]
vals = [int(v) for v in sys.argv[2].split(",")]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dev = torch.device("cuda:0")


def fill(n, tid, lo, hi):
    return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, 0,
                           gen.DIST_UNIFORM, lo, hi)


NV, ND, M = 1 << 28, 1 << 26, 8192
x_v = fill(NV, gen.TID_X, -1.0, 1.0)
y_v = torch.empty(NV, device=dev)
x_d, y_d = fill(ND, gen.TID_X, 0.0, 1.0), fill(ND, gen.TID_Y, 0.0, 2.0)
A = fill(M * M, gen.TID_A, 0.0, 3.0).view(M, M)
gx, gy = fill(M, gen.TID_X, 0.0, 1.0), fill(M, gen.TID_Y, 0.0, 2.0)
go, ra, rd = torch.empty(M, device=dev), torch.empty(1, device=dev), torch.empty(1, device=dev)
ws_a, ws_d = lift.Workspace(NV, dev), lift.Workspace(ND, dev)
BYTES = 12 * NV + 8 * ND + 4 * (M * M + 3 * M)


def step():
    lift.scal(3.0, x_v, out=y_v)
    lift.asum(x_v, out=ra, ws=ws_a)
    lift.dot(x_d, y_d, out=rd, ws=ws_d)
    lift.gemv(A, gx, gy, 1.5, 0.5, out=go)


res = {v: [] for v in vals}
for rep in range(9):
    for v in vals:
        lift.set_variant(knob, v)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K):
            step()
        e.record()
        e.synchronize()
        res[v].append(s.elapsed_time(e) / K)
lift.set_variant(knob, 0)
out = {}
for v in vals:
    ms = sorted(res[v])[4]
    out[f"{knob}={v}"] = {"ms": round(ms, 4), "GB/s": round(BYTES / ms / 1e6, 1),
                          "min_ms": round(min(res[v]), 4), "max_ms": round(max(res[v]), 4)}
print(json.dumps(out))
