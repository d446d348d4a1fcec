"""A/B timing of gemv shapes across liblift builds: python scripts/ab_gemv.py lib1.so ...

Per shape: `reps` launches in one CUDA graph, each on a different copy of A (enough
copies that the rotation exceeds L2), median of 5 replays; plus a hash of y_out's bits
so that variants can be checked bit-identical (every (NT, R, U) must give the same bits)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = [(1024, 8192), (2048, 8192), (4096, 4096), (4096, 8192), (8192, 8192), (8192, 16384),
          (512, 16384), (256, 8192)]


def child(reps=24):
    import torch
    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    dev = torch.device("cuda:0")
    out = {}
    for (m, n) in SHAPES:
        copies = max(2, min(reps, (768 << 20) // (4 * m * n) + 1))
        As = [gen.fill_device(torch.empty(m * n, device=dev), c, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
              for c in range(copies)]
        gx = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
        gy = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
        go = torch.empty(m, device=dev)
        lift.gemv(As[0], gx, gy, 1.5, 0.5, out=go)
        torch.cuda.synchronize()
        h = hashlib.sha1(go.cpu().numpy().tobytes()).hexdigest()[:12]
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    lift.gemv(As[i % copies], gx, gy, 1.5, 0.5, out=go)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(s)
                g.replay()
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / reps * 1e3)
        us = sorted(ts)[2]
        out[f"{m}x{n}"] = {"us": round(us, 2), "GB/s": round(4 * (m * n + n + 2 * m) / us / 1e3, 1),
                           "hash": h}
        del As, g
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child()
        sys.exit(0)
    for lib in sys.argv[1:]:
        env = dict(os.environ, LIFT_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(json.dumps({"lib": os.path.basename(lib)}), r.stdout.strip(), r.stderr[-1500:], flush=True)
