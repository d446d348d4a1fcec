"""Bit-identity of compile-time variant builds: python scripts/variant_bits.py lib1.so lib2.so ...
Each library (same ABI) computes scal/asum/dot/gemv on fixed seeded inputs in its own
subprocess; prints one hash per library — every variant that keeps the canonical order
must print the same hash as the default build."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import torch
    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    dev = torch.device("cuda:0")
    h = hashlib.sha1()

    def fill(n, tid, lo=-1.0, hi=1.0, seed=3):
        return gen.fill_device(torch.empty(n, device=dev), seed, tid, 0, 0, lo, hi)
    for n in (1, 9, 8191, 8192 * 3 + 5, 1 << 20, (1 << 24) + 3):
        x, y = fill(n, 1), fill(n, 2)
        for t in (lift.scal(3.0, x), lift.asum(x), lift.dot(x, y), lift.scal_asum(0.5, x)[1]):
            h.update(t.cpu().numpy().tobytes())
    for m, n in ((300, 2048), (257, 4096), (640, 8192), (33, 16384), (7, 1000), (3, 70000)):
        A = fill(m * n, 3, 0.0, 3.0).view(m, n)
        h.update(lift.gemv(A, fill(n, 1, 0.0, 1.0), fill(m, 2, 0.0, 2.0), 1.5, 0.5).cpu().numpy().tobytes())
    print(h.hexdigest()[:16])


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child()
        sys.exit(0)
    for lib in sys.argv[1:]:
        env = dict(os.environ, LIFT_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(os.path.basename(lib), r.stdout.strip() or r.stderr[-600:], flush=True)
