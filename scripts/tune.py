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
    "ticket_fence": [("acq_rel", "-DLIFT_SC_FENCE=0"), ("sc_fence", "-DLIFT_SC_FENCE=1"),
                     ("release_then_acquire", "-DLIFT_SC_FENCE=2")],
    # Fig. 7a/7b axes: the intra-warp tree in shared memory (toLocal +
    # iterate(split-2 reduce), the paper's lowering) vs the shuffle butterfly — same bits
    "tree": [("shuffle", "-DLIFT_TREE=1"), ("smem_tree", "-DLIFT_TREE=2")],
    # vector width / load path: LDG.256 (default), LDG.128 and scalar via the RUNTIME knob
    # (lift_set_variant LIFT_VAR_LOAD_WIDTH, same build), TMA bulk copies into shared memory
    # for the map (scal) and the reductions (compile-time)
    "load": [("ldg256", "", "load_width=8"), ("ldg128", "", "load_width=4"),
             ("scalar", "", "load_width=1"), ("tma_bulk", "-DLIFT_SCAL_TMA=1 -DLIFT_RED_TMA=1")],
    # gemv toLocal(x) strategies (RUNTIME knob LIFT_VAR_GEMV_X, same build): x through L1
    # widened per use; x fp64 in shared memory + register ring; x fp64 in shared memory +
    # TMA ring of A row segments (warp-specialised producer)
    "gemv_x": [("x_l1", "", "gemv_x=1"), ("x_tma_smem", "", "gemv_x=5"),
               ("x_smem_regring", "", "gemv_x=2"), ("x_smem_tmaring", "", "gemv_x=3"),
               ("x_two_rows", "", "gemv_x=4")],
    # TMA L2 prefetch before the PDL wait and the reductions' chunk order (runtime knobs)
    "prefetch": [("pf_off", "", "prefetch=1"), ("pf_on", "", "prefetch=2")],
    "order": [("ascending", "", "order=1"), ("descending", "", "order=2")],
    # first-wave stagger, ns per 32 KiB a CTA reads (runtime knob LIFT_VAR_STAGGER; default 2)
    "stagger": [("stagger_off", "", "stagger=1"), ("stagger_3ns", "", "stagger=3"),
                ("stagger_4ns", "", "stagger=4"), ("stagger_6ns", "", "stagger=6")],
}


def variants():
    """(name, compile flags, runtime knobs); runtime-only points reuse the default build."""
    vs = [("default", "", "")]
    for axis, pts in SPACE.items():
        for pt in pts:
            name, flags = pt[0], pt[1]
            vs.append((f"{axis}={name}", flags, pt[2] if len(pt) > 2 else ""))
    return vs


def so_path(name, flags):
    return os.path.join(OUT, (name.replace("=", "_") if flags else "default") + ".so")


def build():
    os.makedirs(OUT, exist_ok=True)
    nv = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
          "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
          "-I", os.path.join(ROOT, "include")]
    src = os.path.join(ROOT, "paper_1502_02389_b200", "csrc", "lift.cu")

    def one(v):
        name, flags, _ = v
        so = so_path(name, flags)
        if not flags and name != "default":
            return name, 0, ""
        r = subprocess.run(nv + flags.split() + [src, "-o", so], capture_output=True, text=True)
        return name, r.returncode, r.stderr[-500:]

    with ThreadPoolExecutor(8) as ex:
        for name, rc, err in ex.map(one, variants()):
            print(f"{'ok ' if rc == 0 else 'ERR'} {name} {err if rc else ''}")


def measure(out_path=None):
    ab = os.path.join(ROOT, "scripts", "ab.py")
    results = {}
    for name, flags, knobs in variants():
        so = so_path(name, flags)
        if not os.path.exists(so):
            continue
        env = dict(os.environ, LIFT_LIB=so, LIFT_SET_VARIANTS=knobs)
        r = subprocess.run([sys.executable, ab, "--child"], env=env, capture_output=True, text=True,
                           timeout=600)
        try:
            results[name] = {"flags": flags, "knobs": knobs,
                             **json.loads(r.stdout.strip().splitlines()[-1])}
        except Exception:
            results[name] = {"flags": flags, "knobs": knobs, "error": r.stderr[-800:]}
        print(name, json.dumps(results[name]), flush=True)
    best = {}
    ops = sorted({k for v in results.values() for k in v if k not in ("flags", "knobs", "error")})
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
    if out_path:
        with open(os.path.splitext(out_path)[0] + "_summary.txt", "w") as f:
            f.write(summary(report))


def summary(report):
    """Fixed-width table: us per launch for every variant x op, then the winner per op and
    per axis (the paper's 'chosen by exploring different values empirically')."""
    res = report["results"]
    ops = sorted({k for v in res.values() for k in v if k not in ("flags", "knobs", "error")})
    lines = ["# NEXT-4 variant search (scripts/tune.py): us per launch (CUDA-graph replay of 30 "
             "back-to-back launches, median of 5). One axis varied at a time; every variant "
             "computes the same canonical order except red_k (a different chunk size).",
             "variant".ljust(28) + "".join(o[:11].rjust(12) for o in ops)]
    for n, v in res.items():
        lines.append(n[:27].ljust(28) + "".join(
            (f"{v[o]['us']:.2f}" if o in v else "-").rjust(12) for o in ops))
    lines.append("")
    lines.append("winner per op: " + json.dumps(report["best"]))
    axes = {}
    for n in res:
        if "=" in n:
            axes.setdefault(n.split("=")[0], []).append(n)
    lines.append("")
    lines.append("winner per axis and op (us; default in parentheses):")
    for ax, names in axes.items():
        row = []
        for o in ops:
            c = [(res[n][o]["us"], n.split("=")[1]) for n in names if o in res[n]]
            if c:
                us, w = min(c)
                row.append(f"{o}:{w}({us:.2f}/{res['default'][o]['us']:.2f})")
        lines.append(f"  {ax}: " + "  ".join(row))
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    if sys.argv[1:2] == ["build"]:
        build()
    elif sys.argv[1:2] == ["summary"]:
        with open(sys.argv[2]) as f:
            print(summary(json.load(f)))
    elif sys.argv[1:2] == ["measure"]:
        measure(sys.argv[2] if len(sys.argv) > 2 else None)
    else:
        print(__doc__)
