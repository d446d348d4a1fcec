"""gemv at shapes far from the paper's (documentation of limits): device time per launch,
CUDA-graph replay, median of 5.   python scripts/gemv_shapes.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
out = {}
for (m, n) in [(1, 1 << 24), (16, 1 << 22), (256, 1 << 20), (1 << 24, 8), (1 << 20, 64),
               (1 << 18, 512), (65536, 2048), (8192, 8192)]:
    A = gen.fill_device(torch.empty(m * n, device=dev), 0, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
    x = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
    y = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
    o = torch.empty(m, device=dev)
    s = torch.cuda.Stream(device=dev)
    reps = 5
    with torch.cuda.stream(s):
        lift.gemv(A, x, y, 1.5, 0.5, out=o)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                lift.gemv(A, x, y, 1.5, 0.5, out=o)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / reps * 1e3)
    us = sorted(ts)[2]
    out[f"{m}x{n}"] = {"us": round(us, 2), "GB/s": round(4 * (m * n + n + 2 * m) / us / 1e3, 1)}
    del A
print(json.dumps(out))
