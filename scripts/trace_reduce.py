"""Diagnostic: CTA timeline of one asum (or dot) launch after an L2 flush
(needs build/liblift_trace.so, -DLIFT_TRACE).   python scripts/trace_reduce.py [n] [asum|dot]"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LIFT_LIB"] = os.path.join(ROOT, "build", "liblift_trace.so")
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
op = sys.argv[2] if len(sys.argv) > 2 else "asum"
x = gen.fill_device(torch.empty(n, device="cuda"), 0, 1, 0, 0, -1.0, 1.0)
yv = gen.fill_device(torch.empty(n, device="cuda"), 0, 2, 0, 0, -1.0, 1.0)
ws = lift.Workspace(n, torch.device("cuda"))
r = torch.empty(1, device="cuda")
flush = torch.ones(128 << 20, device="cuda")
def run():
    if op == "dot":
        lift.dot(x, yv, out=r, ws=ws)
    else:
        lift.asum(x, out=r, ws=ws)


for _ in range(3):
    run()
flush.sum()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
nc = (n + lift.CHUNK_ELEMS - 1) // lift.CHUNK_ELEMS
buf = np.zeros(3 * 65536, np.uint64)
lift._lib.lib.lift_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lift._lib.lib.lift_trace_read(buf.ctypes.data, buf.nbytes)
tr = buf[:3 * nc].reshape(nc, 3).astype(np.int64)
t0 = tr[:, 0].min()
start, end, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, tr[:, 2]
fin = (int(buf[3 * 65535]) - t0) / 1e3 if nc < 65535 else None
out = {"n": n, "op": op, "event_us": e0.elapsed_time(e1) * 1e3, "chunks": nc,
       "final_store_us": fin,
       "first_start_us": 0.0, "last_start_us": float(start.max()),
       "last_end_us": float(end.max()), "median_cta_us": float(np.median(end - start)),
       "p10_cta_us": float(np.percentile(end - start, 10)),
       "p90_cta_us": float(np.percentile(end - start, 90)),
       "sms_used": int(len(np.unique(sm))),
       "start_quantiles_us": [float(np.percentile(start, q)) for q in (1, 10, 50, 90, 99)],
       "end_quantiles_us": [float(np.percentile(end, q)) for q in (1, 10, 50, 90, 99)]}
bins = np.arange(0, float(end.max()) + 0.5, 0.5)
out["starts_per_0.5us"] = np.histogram(start, bins)[0].tolist()
out["ends_per_0.5us"] = np.histogram(end, bins)[0].tolist()
print(json.dumps(out))
