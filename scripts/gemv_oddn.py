import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import lift_inputs as gen, paper_1502_02389_b200 as lift
dev = torch.device("cuda:0")
out = {}
for (m, n) in [(8192, 8192), (8192, 8188), (8192, 8190), (8192, 8191), (8192, 8193), (16384, 1001), (16384, 1024)]:
    A = gen.fill_device(torch.empty(m * n, device=dev), 0, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
    x = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
    y = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
    o = torch.empty(m, device=dev)
    s = torch.cuda.Stream(device=dev); reps = 10
    with torch.cuda.stream(s):
        lift.gemv(A, x, y, 1.5, 0.5, out=o); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): lift.gemv(A, x, y, 1.5, 0.5, out=o)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s); g.replay(); e1.record(s); e1.synchronize()
            ts.append(e0.elapsed_time(e1) / reps * 1e3)
    us = sorted(ts)[2]
    out[f"{m}x{n}"] = {"us": round(us, 2), "GB/s": round(4 * m * n / us / 1e3, 1)}
print(json.dumps(out))
