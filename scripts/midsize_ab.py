"""Mid-size reductions back to back (CUDA-graph replay of 30 launches rotating over 4
disjoint slices > L2, median of 5): python scripts/midsize_ab.py  (LIFT_LIB selects the build)"""
import hashlib
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

dev = torch.device("cuda:0")
X = gen.fill_device(torch.empty(1 << 28, device=dev), 0, gen.TID_X, 0, 0, -1.0, 1.0)
Y = gen.fill_device(torch.empty(1 << 28, device=dev), 0, gen.TID_Y, 0, 0, -1.0, 1.0)
ws = lift.Workspace(1 << 26, dev)
r = torch.empty(1, device=dev)
out, h = {}, hashlib.sha1()
for lg in (21, 22, 23, 24, 25):
    n = 1 << lg
    for op in ("asum", "dot"):
        def f(i):
            x, y = X[i << 26:(i << 26) + n], Y[i << 26:(i << 26) + n]
            return lift.asum(x, out=r, ws=ws) if op == "asum" else lift.dot(x, y, out=r, ws=ws)
        for i in range(4):
            h.update(f(i).cpu().numpy().tobytes())
        cs = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(cs):
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for k in range(30):
                    f(k % 4)
            ts = []
            for _ in range(5):
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record(cs)
                g.replay()
                e.record(cs)
                e.synchronize()
                ts.append(s.elapsed_time(e) / 30 * 1e3)
        out[f"{op}_2p{lg}"] = round(sorted(ts)[2], 2)
out["hash"] = h.hexdigest()[:12]
print(json.dumps(out))
