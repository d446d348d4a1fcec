"""How the bench step's schedule affects its time (same kernels, same bytes):
    python scripts/step_ab.py [K]
  seq_events   : the bench.py step (per-op events between kernels)
  seq_plain    : same launches, events only around the K steps
  graph        : K steps captured in one CUDA graph (PDL edges kept)
  2streams     : scal->asum on one stream, dot->gemv on another (the ops are independent)
  4streams     : each op on its own stream, joined per step
  order_*      : other sequential orders
Prints ms/step and GB/s for each (median of 5 repetitions of K steps)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402
for _kv in filter(None, os.environ.get("LIFT_SET_VARIANTS", "").split(",")):
    lift.set_variant(_kv.split("=")[0], int(_kv.split("=")[1]))  # NEXT-4 runtime knobs

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)


def fill(n, tid, lo, hi):
    return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, 0,
                           gen.DIST_UNIFORM, lo, hi)


NV, ND, M = 1 << 28, 1 << 26, 8192
x_v = fill(NV, gen.TID_X, -1.0, 1.0)
y_v = torch.empty(NV, device=dev)
x_d = fill(ND, gen.TID_X, 0.0, 1.0)
y_d = fill(ND, gen.TID_Y, 0.0, 2.0)
A = fill(M * M, gen.TID_A, 0.0, 3.0).view(M, M)
gx = fill(M, gen.TID_X, 0.0, 1.0)
gy = fill(M, gen.TID_Y, 0.0, 2.0)
go = torch.empty(M, device=dev)
ra = torch.empty(1, device=dev)
rd = torch.empty(1, device=dev)
ws_a = lift.Workspace(NV, dev)
ws_d = lift.Workspace(ND, dev)
BYTES = 12 * NV + 8 * ND + 4 * (M * M + 3 * M)
ops = {"scal": lambda: lift.scal(3.0, x_v, out=y_v),
       "asum": lambda: lift.asum(x_v, out=ra, ws=ws_a),
       "dot": lambda: lift.dot(x_d, y_d, out=rd, ws=ws_d),
       "gemv": lambda: lift.gemv(A, gx, gy, 1.5, 0.5, out=go)}
main = torch.cuda.current_stream(dev)
side = [torch.cuda.Stream(dev) for _ in range(4)]
ws_side = [lift.Workspace(NV, dev) for _ in range(4)]


def seq(order, events=False):
    def f(evs=None):
        for i, o in enumerate(order):
            if events:
                evs[i].record(main)
            ops[o]()
        if events:
            evs[len(order)].record(main)
    return f


def streams(groups):
    """groups: list of op lists; each list runs on its own stream; joined at the end."""
    def f(evs=None):
        fork = torch.cuda.Event()
        fork.record(main)
        joins = []
        for gi, g in enumerate(groups):
            s = side[gi]
            s.wait_event(fork)
            with torch.cuda.stream(s):
                for o in g:
                    if o == "asum":
                        lift.asum(x_v, out=ra, ws=ws_side[gi])
                    elif o == "dot":
                        lift.dot(x_d, y_d, out=rd, ws=ws_side[gi])
                    else:
                        ops[o]()
            e = torch.cuda.Event()
            e.record(s)
            joins.append(e)
        for e in joins:
            main.wait_event(e)
    return f


def timeit(step, events=False, reps=5):
    res = []
    for _ in range(reps):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
        for _ in range(3):
            step(evs[0])
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(main)
        for k in range(K):
            step(evs[k])
        e.record(main)
        torch.cuda.synchronize()
        res.append(s.elapsed_time(e) / K)
    res.sort()
    return res[len(res) // 2]


def graph_time(step, reps=5):
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(dev)
    with torch.cuda.stream(cs):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(K):
                step()
    res = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(cs)
        g.replay()
        e.record(cs)
        e.synchronize()
        res.append(s.elapsed_time(e) / K)
    res.sort()
    return res[len(res) // 2]


out = {}
base = ["scal", "asum", "dot", "gemv"]
out["seq_events"] = timeit(seq(base, True), True)
out["seq_plain"] = timeit(seq(base))
out["graph"] = graph_time(seq(base))
for order in (["scal", "gemv", "asum", "dot"], ["gemv", "scal", "dot", "asum"],
              ["dot", "scal", "gemv", "asum"], ["scal", "dot", "asum", "gemv"]):
    out["order_" + ",".join(order)] = timeit(seq(order))
out["2streams"] = timeit(streams([["scal", "asum"], ["dot", "gemv"]]))
out["2streams_b"] = timeit(streams([["scal"], ["asum", "dot", "gemv"]]))
out["4streams"] = timeit(streams([["scal"], ["asum"], ["dot"], ["gemv"]]))
for k in ("scal", "asum", "dot", "gemv"):
    out["alone_" + k] = timeit(seq([k]))
print(json.dumps({k: {"ms": round(v, 4), "GB/s": round(BYTES / v / 1e6, 1)} if not k.startswith("alone")
                  else {"ms": round(v, 4)} for k, v in out.items()}, indent=1))
