"""Cost of the NEXT-1 in-kernel exchange code path at p = 1 (measurable on one GPU): the
fused-all-gather gemv (lift_gemv_allgather: PEERS kernel — per-CTA block count, flag
publish and wait) and the fused all-reduce asum/dot vs the plain calls: `reps` calls
captured in one CUDA graph (eager Python launches would measure the binding's overhead),
mean per call, median of 5 replays.  (At p = 1 a replayed epoch only re-publishes the same
flag value, so the frozen epochs of a graph are harmless.)
    python scripts/xchg_p1.py  (prints one JSON line)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402
from paper_1502_02389_b200 import dist as ldist  # noqa: E402

dev = torch.device("cuda:0")
ex = ldist.PeerExchange(device=dev)


def timed(f, reps=40):
    cs = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(cs):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(reps):
                f()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(cs)
            g.replay()
            e.record(cs)
            e.synchronize()
            ts.append(s.elapsed_time(e) / reps * 1e3)
    return round(sorted(ts)[2], 2)


out = {"note": "p = 1: the exchange code path without a peer; CUDA-graph replay, us per call"}
for m, n in ((8192, 8192), (8192, 16384), (4096, 4096)):
    A = gen.fill_device(torch.empty(m * n, device=dev), 0, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
    x = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
    y = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
    o = torch.empty(m, device=dev)
    plain = timed(lambda: lift.gemv(A, x, y, 1.5, 0.5, out=o))
    fused = timed(lambda: ex.gemv(A, x, y, 1.5, 0.5, m, 0))
    same = torch.equal(ex.gemv(A, x, y, 1.5, 0.5, m, 0).view(torch.int32),
                       lift.gemv(A, x, y, 1.5, 0.5).view(torch.int32))
    out[f"gemv {m}x{n}"] = {"plain_us": plain, "fused_p1_us": fused,
                            "overhead_us": round(fused - plain, 2), "same_bits": bool(same)}
for nlog in (24, 26):
    N = 1 << nlog
    xv = gen.fill_device(torch.empty(N, device=dev), 0, gen.TID_X, 0, 0, -1.0, 1.0)
    yv = gen.fill_device(torch.empty(N, device=dev), 0, gen.TID_Y, 0, 0, -1.0, 1.0)
    ws = lift.Workspace(N, dev)
    r = torch.empty(1, device=dev)
    out[f"asum 2^{nlog}"] = {"plain_us": timed(lambda: lift.asum(xv, out=r, ws=ws)),
                             "fused_p1_us": timed(lambda: ex.asum(xv, out=r, ws=ws))}
    out[f"dot 2^{nlog}"] = {"plain_us": timed(lambda: lift.dot(xv, yv, out=r, ws=ws)),
                            "fused_p1_us": timed(lambda: ex.dot(xv, yv, out=r, ws=ws))}
ex.check()
ex.close()
print(json.dumps(out))
