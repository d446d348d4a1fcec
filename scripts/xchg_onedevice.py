"""NEXT-1 on one device: two "ranks" as two concurrent streams of one process, sharing
their exchange buffers directly (no IPC), each reducing half of the operand with the
combine fused into the kernel (lift_asum_allreduce / lift_dot_allreduce).  Compared with
the single-rank call over the whole operand, the difference is the in-kernel exchange
(flag publish, wait, fold of p partials) plus the cost of splitting one launch in two.
Peer stores here go to the same device's memory; across GPUs they cross NVLink.

    python scripts/xchg_onedevice.py   (prints one JSON line)"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402
from paper_1502_02389_b200._lib import check, lib  # noqa: E402

dev = torch.device("cuda:0")
P = 2


def run(n_total, reps=50, op="asum"):
    n = n_total // P
    x = gen.fill_device(torch.empty(n_total, device=dev), 0, gen.TID_X, 0, 0, -1.0, 1.0)
    y = gen.fill_device(torch.empty(n_total, device=dev), 0, gen.TID_Y, 0, 0, -1.0, 1.0)
    bufs = []
    for _ in range(P):
        b = ctypes.c_void_p()
        check(lib.lift_xchg_create(P, ctypes.byref(b)))
        bufs.append(b.value)
    peers = torch.tensor(bufs, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = [lift.Workspace(n, dev) for _ in range(P)]
    res = torch.empty(P, device=dev)
    streams = [torch.cuda.Stream(device=dev) for _ in range(P)]
    wsf = lift.Workspace(n_total, dev)
    rf = torch.empty(1, device=dev)
    epoch = [0]

    def fused():
        epoch[0] += 1
        for r in range(P):
            s = streams[r]
            xs, ys = x[r * n:(r + 1) * n], y[r * n:(r + 1) * n]
            if op == "asum":
                check(lib.lift_asum_allreduce(n, xs.data_ptr(), res[r:r + 1].data_ptr(), ws[r].ptr,
                                              ws[r].nbytes, peers.data_ptr(), P, r, epoch[0],
                                              err.data_ptr(), s.cuda_stream))
            else:
                check(lib.lift_dot_allreduce(n, xs.data_ptr(), ys.data_ptr(), res[r:r + 1].data_ptr(),
                                             ws[r].ptr, ws[r].nbytes, peers.data_ptr(), P, r,
                                             epoch[0], err.data_ptr(), s.cuda_stream))

    def single():
        if op == "asum":
            lift.asum(x, out=rf, ws=wsf)
        else:
            lift.dot(x, y, out=rf, ws=wsf)

    def timed(fn, multi):
        main = torch.cuda.current_stream(dev)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(main)
        for s in streams:
            s.wait_event(e0)
        for _ in range(reps):
            if multi:
                fn()
            else:
                with torch.cuda.stream(streams[0]):
                    fn()
        ends = []
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            ends.append(ev)
        for ev in ends:
            main.wait_event(ev)
        e1.record(main)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    t_single = timed(single, False)
    t_fused = timed(fused, True)
    torch.cuda.synchronize()
    same = bool(torch.equal(res[0:1], res[1:2]))
    for b in bufs:
        lib.lift_xchg_destroy(b)
    return {"n_total": n_total, "single_us": round(t_single, 2), "fused_2rank_us": round(t_fused, 2),
            "overhead_us": round(t_fused - t_single, 2), "ranks_agree": same,
            "error_flag": int(err.item())}


out = {"note": "two ranks = two concurrent streams on one B200 (exchange through the same "
               "device's memory); single = one launch over the whole operand; back-to-back "
               "launches, mean per call"}
for k in (20, 24, 26):
    out[f"asum_2^{k}"] = run(1 << k, op="asum")
    out[f"dot_2^{k}"] = run(1 << k, op="dot")
print(json.dumps(out))
