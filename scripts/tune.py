"""NEXT-4: bounded search over the B200 variant space of the hot path.

The paper derives device-specific variants of the same expression (Fig. 7a/7b/7c,
P:1001-1027; split sizes and vector widths "chosen by exploring different values
empirically") and sketches an automatic search.  Here the
variant space is the kernels' compile-time knobs; each point is a separate build of
liblift.so (same ABI), timed on the device with scripts/ab.py's harness.

    python scripts/tune.py build             # here (CPU): nvcc every variant into build/tune/
    python scripts/tune.py measure [out]     # on the B200: time every variant, rank per op

Knobs that change the canonical summation order (LIFT_RED_K) produce a different —
equally valid, still deterministic — reduction order (reading R2/R5); the chosen
defaults live in csrc/canon.h and lift.cu.
"""
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "tune")

# (name, -D flags) — one axis at a time around the defaults, plus a few joint points
SPACE = {
    "red_k": [("k2", "-DLIFT_RED_K=2"), ("k4", "-DLIFT_RED_K=4"),
              ("k8", "-DLIFT_RED_K=8 -DLIFT_RED_G=128"),
              ("k16", "-DLIFT_RED_K=16 -DLIFT_RED_G=64")],
    "asum_acc": [("asum_f32", "-DLIFT_ASUM_ACC=float"), ("asum_f64", "-DLIFT_ASUM_ACC=double")],
    "dot_acc": [("dot_f64", "-DLIFT_DOT_ACC=double"), ("dot_f32", "-DLIFT_DOT_ACC=float")],
    "gemv_b": [("g_b4m4", "-DLIFT_GEMV_B=4 -DLIFT_GEMV_MINB=4"),
               ("g_b2m6", "-DLIFT_GEMV_B=2 -DLIFT_GEMV_MINB=6"),
               ("g_b8m2", "-DLIFT_GEMV_B=8 -DLIFT_GEMV_MINB=2"),
               ("g_b4m3", "-DLIFT_GEMV_B=4 -DLIFT_GEMV_MINB=3")],
    "grid": [("nonpersistent", "-DLIFT_PERSISTENT=0"), ("persistent", "-DLIFT_PERSISTENT=1")],
    "scal_tile": [("s1024x1", "-DLIFT_SCAL_T=1024 -DLIFT_SCAL_U=1"),
                  ("s512x1", "-DLIFT_SCAL_T=512 -DLIFT_SCAL_U=1"),
                  ("s256x2", "-DLIFT_SCAL_T=256 -DLIFT_SCAL_U=2"),
                  ("s256x4", "-DLIFT_SCAL_T=256 -DLIFT_SCAL_U=4")],
    "pdl": [("pdl_on", "-DLIFT_PDL=1"), ("pdl_off", "-DLIFT_PDL=0")],
    "ticket_fence": [("acq_rel", "-DLIFT_SC_FENCE=0"), ("sc_fence", "-DLIFT_SC_FENCE=1")],
}


def variants():
    vs = [("default", "")]
    for axis, pts in SPACE.items():
        for name, flags in pts:
            vs.append((f"{axis}={name}", flags))
    return vs


def build():
    os.makedirs(OUT, exist_ok=True)
    nv = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
          "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
          "-I", os.path.join(ROOT, "include")]
    src = os.path.join(ROOT, "paper_1502_02389_b200", "csrc", "lift.cu")

    def one(v):
        name, flags = v
        so = os.path.join(OUT, name.replace("=", "_") + ".so")
        r = subprocess.run(nv + flags.split() + [src, "-o", so], capture_output=True, text=True)
        return name, r.returncode, r.stderr[-500:]

    with ThreadPoolExecutor(8) as ex:
        for name, rc, err in ex.map(one, variants()):
            print(f"{'ok ' if rc == 0 else 'ERR'} {name} {err if rc else ''}")


def measure(out_path=None):
    ab = os.path.join(ROOT, "scripts", "ab.py")
    results = {}
    for name, flags in variants():
        so = os.path.join(OUT, name.replace("=", "_") + ".so")
        if not os.path.exists(so):
            continue
        env = dict(os.environ, LIFT_LIB=so)
        r = subprocess.run([sys.executable, ab, "--child"], env=env, capture_output=True, text=True,
                           timeout=600)
        try:
            results[name] = {"flags": flags, **json.loads(r.stdout.strip().splitlines()[-1])}
        except Exception:
            results[name] = {"flags": flags, "error": r.stderr[-800:]}
        print(name, json.dumps(results[name]), flush=True)
    best = {}
    ops = sorted({k for v in results.values() for k in v if k not in ("flags", "error")})
    for op in ops:
        cand = [(v[op]["us"], n) for n, v in results.items() if op in v]
        if cand:
            us, n = min(cand)
            best[op] = {"variant": n, "us": us, "default_us": results["default"][op]["us"]}
    report = {"note": "each variant = one liblift.so build; times: median of 5 rounds of 30 "
                      "back-to-back launches (scripts/ab.py)", "results": results, "best": best}
    if out_path:
        with open(out_path, "w") as f:
            json.dump(report, f, indent=1)
    print(json.dumps(best, indent=1))


if __name__ == "__main__":
    if sys.argv[1:2] == ["build"]:
        build()
    elif sys.argv[1:2] == ["measure"]:
        measure(sys.argv[2] if len(sys.argv) > 2 else None)
    else:
        print(__doc__)
