"""C3-style size sweep: scal / asum / dot at n = 2^16 .. 2^28 (and gemv at the paper's
sizes), device time per launch from CUDA-graph replays (no Python launch overhead),
L2 flushed between replays for sizes that would otherwise stay L2-resident.

    python scripts/sweep.py > profiles/<round>/sweep.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
PEAK = 6451.8


def fill(n, tid, lo, hi):
    return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, 0, 0, lo, hi)


# L2 flush by READING 512 MiB (> 4x L2): leaves only clean lines behind, so the timed
# launch does not pay for write-backs of a flush buffer (zero-filling one would).
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)


def time_op(fn, nbytes, reps=20, flush_l2=True):
    """Median over `reps` of one graph-replayed launch; L2 flushed (by reads) before each.
    A single launch includes its ramp-up and drain, so these are lower than the
    back-to-back figures of scripts/ab.py and bench.py."""
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        fn()  # warm (workspace, occupancy cache)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    ts = []
    for _ in range(reps):
        if flush_l2:
            flush.sum()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    us = ts[len(ts) // 2] * 1e3
    gbs = nbytes / (us * 1e-6) / 1e9
    return {"us": round(us, 2), "GB/s": round(gbs, 1), "frac_measured": round(gbs / PEAK, 3),
            "frac_8TBs": round(gbs / 8000, 3)}


out = {"note": "device time per launch, CUDA graph replay, L2 flushed before each launch, "
               "median of 20; HBM roofline denominators: 6451.8 GB/s measured, 8 TB/s nominal"}
x = fill(1 << 28, 1, -1.0, 1.0)
y = fill(1 << 28, 2, 0.0, 2.0)
yo = torch.empty(1 << 28, dtype=torch.float32, device=dev)
r = torch.empty(1, dtype=torch.float32, device=dev)
ws = lift.Workspace(1 << 28, dev)
for k in range(16, 29, 2):
    n = 1 << k
    xs, ys, yos = x[:n], y[:n], yo[:n]
    out[f"scal_2^{k}"] = time_op(lambda: lift.scal(3.0, xs, out=yos), 8 * n)
    out[f"asum_2^{k}"] = time_op(lambda: lift.asum(xs, out=r, ws=ws), 4 * n)
    out[f"dot_2^{k}"] = time_op(lambda: lift.dot(xs, ys, out=r, ws=ws), 8 * n)
del x, y, yo
# C5: dot over 2^31 elements on one GPU (16 GiB of inputs), as one launch
big_x = fill(1 << 31, 1, 0.0, 1.0)
big_y = fill(1 << 31, 2, 0.0, 2.0)
wsb = lift.Workspace(1 << 31, dev)
out["dot_2^31"] = time_op(lambda: lift.dot(big_x, big_y, out=r, ws=wsb), 8 << 31, reps=5,
                          flush_l2=False)
del big_x, big_y
for (m, n) in [(4096, 4096), (8192, 8192), (8192, 16384)]:
    A = fill(m * n, 3, 0.0, 3.0).view(m, n)
    gx, gy = fill(n, 1, 0.0, 1.0), fill(m, 2, 0.0, 2.0)
    go = torch.empty(m, dtype=torch.float32, device=dev)
    out[f"gemv_{m}x{n}"] = time_op(lambda: lift.gemv(A, gx, gy, 1.5, 0.5, out=go),
                                   4 * (m * n + n + 2 * m))
    del A
print(json.dumps(out, indent=1))
