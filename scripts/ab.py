"""A/B timing of liblift builds: python scripts/ab.py lib1.so [lib2.so ...]

Each library (same ABI, different compile-time tuning) runs in its own subprocess
(LIFT_LIB=...).  Per op: `reps` back-to-back launches captured in one CUDA graph
(no Python launch overhead), median over 5 interleaved replays; operands >= 256 MiB
exceed L2 except the small asum_2p20 case (L2-resident by design: latency).
Prints one JSON line per library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(reps=30):
    import torch
    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    dev = torch.device("cuda:0")
    for kv in filter(None, os.environ.get("LIFT_SET_VARIANTS", "").split(",")):
        k, v = kv.split("=")
        lift.set_variant(k, int(v))  # NEXT-4 runtime knobs (same build)

    def fill(n, tid, lo, hi):
        return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, 0, 0, lo, hi)

    x = fill(1 << 28, 1, -1.0, 1.0)
    y = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    dx = fill(1 << 26, 1, 0.0, 1.0)
    dy = fill(1 << 26, 2, 0.0, 2.0)
    A = fill(8192 * 8192, 3, 0.0, 3.0).view(8192, 8192)
    A2 = fill(8192 * 16384, 3, 0.0, 3.0).view(8192, 16384)
    gx = fill(8192, 1, 0.0, 1.0)
    gx2 = fill(16384, 1, 0.0, 1.0)
    gy = fill(8192, 2, 0.0, 2.0)
    go = torch.empty(8192, dtype=torch.float32, device=dev)
    r = torch.empty(1, dtype=torch.float32, device=dev)
    ws = lift.Workspace(1 << 28, dev)
    bs_s = fill(4 << 20, 1, 10.0, 200.0)
    bs_c = torch.empty(4 << 20, dtype=torch.float32, device=dev)
    bs_p = torch.empty(4 << 20, dtype=torch.float32, device=dev)
    def rot(f, k=4):
        state = [0]

        def g():
            f(state[0] % k)
            state[0] += 1
        return g

    ops = {
        "scal_2p28": (lambda: lift.scal(3.0, x, out=y), 8 << 28),
        "asum_2p28": (lambda: lift.asum(x, out=r, ws=ws), 4 << 28),
        "dot_2p26": (lambda: lift.dot(dx, dy, out=r, ws=ws), 8 << 26),
        "gemv_8192": (lambda: lift.gemv(A, gx, gy, 1.5, 0.5, out=go), 4 * (8192 * 8192 + 3 * 8192)),
        "gemv_8192x16384": (lambda: lift.gemv(A2, gx2, gy, 1.5, 0.5, out=go),
                            4 * (8192 * 16384 + 16384 + 2 * 8192)),
        "asum_2p20": (lambda: lift.asum(x[:1 << 20], out=r, ws=ws), 4 << 20),
        # mid sizes: rotate over 4 disjoint slices so no launch finds its data in L2
        "asum_2p24": (rot(lambda i: lift.asum(x[i << 26:(i << 26) + (1 << 24)], out=r, ws=ws)),
                      4 << 24),
        "dot_2p24": (rot(lambda i: lift.dot(x[i << 26:(i << 26) + (1 << 24)],
                                            y[i << 26:(i << 26) + (1 << 24)], out=r, ws=ws)),
                     8 << 24),
        "scal_asum_2p28": (lambda: lift.scal_asum(3.0, x, out=y, result=r, ws=ws), 8 << 28),
        "bs_4M": (lambda: lift.blackscholes(bs_s, 100.0, 0.05, 0.2, 1.0, call=bs_c, put=bs_p),
                  12 * (4 << 20)),
    }
    out = {}
    samples = {name: [] for name in ops}
    graphs = {}
    cs = torch.cuda.Stream(device=dev)
    for name, (fn, _) in ops.items():  # warm, then capture `reps` launches per op
        with torch.cuda.stream(cs):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for _ in range(reps):
                    fn()
        graphs[name] = g
    torch.cuda.synchronize()
    for _ in range(5):  # rounds interleaved across ops; each = one replay of `reps` launches
        for name in ops:
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            graphs[name].replay()
            e.record()
            e.synchronize()
            samples[name].append(s.elapsed_time(e) / reps)
    for name, (fn, nbytes) in ops.items():
        ts = sorted(samples[name])
        med = ts[len(ts) // 2]
        out[name] = {"us": round(med * 1e3, 2), "GB/s": round(nbytes / (med * 1e-3) / 1e9, 1),
                     "spread%": round(100 * (ts[-1] - ts[0]) / med, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child()
        sys.exit(0)
    for lib in sys.argv[1:]:
        env = dict(os.environ, LIFT_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True,
                           text=True)
        print(json.dumps({"lib": os.path.basename(lib)}), r.stdout.strip(), r.stderr[-2000:],
              flush=True)
