"""Mid-size back-to-back launches on one stream vs round-robin over 4 streams (independent
calls, separate workspaces): how much of a launch's fixed cost is the dependent-launch
chain.  python scripts/midsize_streams.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import lift_inputs as gen  # noqa: E402
import paper_1502_02389_b200 as lift  # noqa: E402

dev = torch.device("cuda:0")
N = 1 << 24
xs = [gen.fill_device(torch.empty(N, device=dev), i, gen.TID_X, 0, 0, -1.0, 1.0) for i in range(4)]
ys = [gen.fill_device(torch.empty(N, device=dev), i, gen.TID_Y, 0, 0, -1.0, 1.0) for i in range(4)]
A = [gen.fill_device(torch.empty(4096 * 4096, device=dev), i, gen.TID_A, 0, 0, 0.0, 3.0).view(4096, 4096)
     for i in range(4)]
gx = gen.fill_device(torch.empty(4096, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
gy = gen.fill_device(torch.empty(4096, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
streams = [torch.cuda.Stream(dev) for _ in range(4)]
wss = [lift.Workspace(N, dev) for _ in range(4)]
outs = [torch.empty(4096, device=dev) for _ in range(4)]
R = 40
ops = {"asum_2p24": lambda i, ws: lift.asum(xs[i], ws=ws),
       "dot_2p24": lambda i, ws: lift.dot(xs[i], ys[i], ws=ws),
       "gemv_4096": lambda i, ws: lift.gemv(A[i], gx, gy, 1.5, 0.5, out=outs[i])}
res = {}
for name, f in ops.items():
    for mode in ("1stream", "4streams"):
        ts = []
        for rep in range(5):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            for st in streams:
                st.wait_stream(torch.cuda.current_stream())
            for k in range(R):
                i = k % 4
                if mode == "1stream":
                    f(i, wss[0])
                else:
                    with torch.cuda.stream(streams[i]):
                        f(i, wss[i])
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) / R * 1e3)
        res[f"{name} {mode}"] = round(sorted(ts)[2], 2)
print(json.dumps(res))
