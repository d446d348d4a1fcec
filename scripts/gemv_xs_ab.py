"""A/B of gemv's x strategies (LIFT_VAR_GEMV_X: 1 = x through L1, widened per use;
2 = x staged once per CTA as fp64 in shared memory) over shapes, in one process per
library: python scripts/gemv_xs_ab.py [lib1.so ...]  (default: the in-tree liblift.so).

Per (shape, variant): `reps` launches in one CUDA graph, each on a different copy of A
(rotation > L2), median of 5 replays, plus a hash of y_out's bits: both variants must
give identical bits (same canonical order)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = [(8192, 8192), (4096, 4096), (8192, 16384), (1024, 8192), (2048, 8192), (512, 8192),
          (256, 8192), (4096, 8192), (8192, 2048), (16384, 4096), (8192, 24576), (2048, 2048),
          (300, 8192)]


def child(reps=24):
    import torch
    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    dev = torch.device("cuda:0")
    for kv in filter(None, os.environ.get("LIFT_SET_VARIANTS", "").split(",")):
        lift.set_variant(kv.split("=")[0], int(kv.split("=")[1]))  # other knobs, fixed
    shapes = SHAPES
    if os.environ.get("AB_SHAPES"):
        shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ["AB_SHAPES"].split(",")]
    out = {}
    for (m, n) in shapes:
        copies = max(2, min(reps, (768 << 20) // (4 * m * n) + 1))
        As = [gen.fill_device(torch.empty(m * n, device=dev), c, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
              for c in range(copies)]
        gx = gen.fill_device(torch.empty(n, device=dev), 0, gen.TID_X, 0, 0, 0.0, 1.0)
        gy = gen.fill_device(torch.empty(m, device=dev), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
        go = torch.empty(m, device=dev)
        row = {}
        knob = os.environ.get("AB_KNOB", "gemv_x")
        vals = tuple(int(v) for v in os.environ.get("AB_VARS", "1,2,3").split(","))
        graphs, hashes = {}, {}
        s = torch.cuda.Stream(device=dev)
        for var in vals:  # capture one graph per variant (the knob is read at launch)
            lift.set_variant(knob, var)
            go.fill_(float("nan"))
            lift.gemv(As[0], gx, gy, 1.5, 0.5, out=go)
            torch.cuda.synchronize()
            hashes[var] = hashlib.sha1(go.cpu().numpy().tobytes()).hexdigest()[:12]
            with torch.cuda.stream(s):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for i in range(reps):
                        lift.gemv(As[i % copies], gx, gy, 1.5, 0.5, out=go)
            graphs[var] = g
        ts = {v: [] for v in vals}
        with torch.cuda.stream(s):  # replay launches on the current stream
            for _ in range(7):  # replays interleaved across variants: drift hits all alike
                for var in vals:
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record(s)
                    graphs[var].replay()
                    e1.record(s)
                    e1.synchronize()
                    ts[var].append(e0.elapsed_time(e1) / reps * 1e3)
        for var in vals:
            us = sorted(ts[var])[3]
            row[f"v{var}"] = {"us": round(us, 2),
                              "GB/s": round(4 * (m * n + n + 2 * m) / us / 1e3, 1), "hash": hashes[var]}
        del graphs
        row["same_bits"] = len({row[k]["hash"] for k in row}) == 1
        out[f"{m}x{n}"] = row
        del As
        print(f"{m}x{n}", json.dumps(row), file=sys.stderr, flush=True)
    lift.set_variant(os.environ.get("AB_KNOB", "gemv_x"), 0)
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child()
        sys.exit(0)
    libs = sys.argv[1:] or [os.path.join(ROOT, "paper_1502_02389_b200", "liblift.so")]
    for lib in libs:
        env = dict(os.environ, LIFT_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(json.dumps({"lib": os.path.basename(lib)}), r.stdout.strip(), r.stderr[-3000:], flush=True)
