"""Throughput on misaligned operands (slices at float offsets 1, 4 from a 256-B aligned
base): back-to-back graph replays, median of 5.   python scripts/misaligned.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
n = 1 << 26
bx = gen.fill_device(torch.empty(n + 64, device=dev), 0, gen.TID_X, 0, 0, -1.0, 1.0)
by = gen.fill_device(torch.empty(n + 64, device=dev), 0, gen.TID_Y, 0, 0, -1.0, 1.0)
bo = torch.empty(n + 64, device=dev)
r = torch.empty(1, device=dev)
m, k = 4096, 8192
bA = gen.fill_device(torch.empty(m * k + 64, device=dev), 0, gen.TID_A, 0, 0, 0.0, 3.0)


def timed(fn, nbytes, reps=20):
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / reps * 1e3)
    us = sorted(ts)[2]
    return {"us": round(us, 2), "GB/s": round(nbytes / us / 1e3, 1)}


out = {}
for off in (0, 1, 4):
    x, y, o = bx[off:off + n], by[off:off + n], bo[off:off + n]
    out[f"asum_off{off}"] = timed(lambda: lift.asum(x, out=r), 4 * n)
    out[f"dot_off{off}"] = timed(lambda: lift.dot(x, y, out=r), 8 * n)
    out[f"scal_off{off}"] = timed(lambda: lift.scal(3.0, x, out=o), 8 * n)
    A = bA[off:off + m * k].view(m, k)
    gx = bx[off:off + k]
    out[f"gemv_off{off}"] = timed(lambda: lift.gemv(A, gx, by[:m], 1.5, 0.5, out=bo[:m]), 4 * m * k)
print(json.dumps(out))
