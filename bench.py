"""bench.py — throughput of the paper's BLAS hot path on B200 (driver contract).

One STEP = one pass of every §8(a) row over one batch of synthetic input, per rank:
    scal  y = 3*x,            n = 2^28   (BASELINE configs[2], Fig. 3's mul3)
    asum  sum|x|,             n = 2^28   (configs[2])
    dot   sum x*y,            n = 2^26   (configs[1], large case)
    gemv  1.5*A@x + 0.5*y,    8192 x 8192 rows per rank (configs[3])
  + X1 at N > 1: all-gather of the asum/dot fp64 partials + lift_combine, and
    all-gather of the gemv y slices (weak scaling: rank r owns global slice r).
metric = achieved HBM GB/s = algorithmic bytes of the step
         / device time.  Every operand is >= 256 MiB > the 126 MB L2, so no flush.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lift|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_VEC = 1 << 28      # scal / asum
N_DOT = 1 << 26      # dot
GEMV_M = 8192        # rows per rank
GEMV_N = 8192
ALPHA_SCAL = 3.0
ALPHA, BETA = 1.5, 0.5
NOMINAL_HBM = 8000.0  # GB/s, BASELINE.json's denominator (nominal)

OPS = tuple(os.environ.get("LIFT_STEP_ORDER", "scal,asum,dot,gemv").split(","))


def op_bytes(world: int = 1) -> dict:
    """Algorithmic bytes per launch (per rank): what the op must move."""
    return {
        "scal": 8 * N_VEC,                                  # read x + write y
        "asum": 4 * N_VEC,                                  # read x
        "dot": 8 * N_DOT,                                   # read x, y
        "gemv": 4 * (GEMV_M * GEMV_N + GEMV_N + 2 * GEMV_M),  # A, x, y in, y_out
    }


def op_elems() -> dict:
    """Elements each op processes per launch (per rank): vector elements, dot pairs, A entries."""
    return {"scal": N_VEC, "asum": N_VEC, "dot": N_DOT, "gemv": GEMV_M * GEMV_N}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """Per-launch dram bytes from the committed ncu --set full capture, if present."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 <= t <= t1] or [r for (_, r) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[2:]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------- oracle arm
def oracle_sample(frac_shift: int):
    """Host inputs for a bounded sample of one step: every op at 1/2^frac_shift size."""
    import lift_inputs as gen
    ns, nd, gm = N_VEC >> frac_shift, N_DOT >> frac_shift, max(1, GEMV_M >> frac_shift)
    return {
        "x": gen.host(ns, 0, gen.TID_X),
        "dx": gen.host(nd, 0, gen.TID_X, lo=0.0, hi=1.0),
        "dy": gen.host(nd, 0, gen.TID_Y, lo=0.0, hi=2.0),
        "A": gen.host(gm * GEMV_N, 0, gen.TID_A, lo=0.0, hi=3.0).reshape(gm, GEMV_N),
        "gx": gen.host(GEMV_N, 0, gen.TID_X, lo=0.0, hi=1.0),
        "gy": gen.host(gm, 0, gen.TID_Y, lo=0.0, hi=2.0),
        "bytes": 12 * ns + 8 * nd + 4 * (gm * GEMV_N + GEMV_N + 2 * gm),
        "desc": (f"one step at 1/{1 << frac_shift} size: scal+asum n=2^{28 - frac_shift}, "
                 f"dot n=2^{26 - frac_shift}, gemv {gm}x{GEMV_N}"),
    }


def oracle_step(s):
    import oracle
    oracle.scal(ALPHA_SCAL, s["x"])
    oracle.asum(s["x"])
    oracle.dot(s["dx"], s["dy"])
    oracle.gemv(s["A"], s["gx"], s["gy"], ALPHA, BETA)


def oracle_step_cores(s, pool, k):
    """The same oracle functions run concurrently on k contiguous shards of every operand
    (fixed 2^16-element-aligned boundaries, partials combined in shard order; the ctypes
    calls release the GIL).  Timing only: SURVEY §8(d) asks for the oracle on all cores."""
    import oracle

    def cuts(n):
        g = 1 << 16
        step = max(g, (n + k * g - 1) // (k * g) * g)  # ceil(n / k), rounded up to 2^16
        return [(a, min(n, a + step)) for a in range(0, n, step)]
    jobs = [pool.submit(oracle.scal, ALPHA_SCAL, s["x"][a:b]) for a, b in cuts(len(s["x"]))]
    jobs += [pool.submit(oracle.asum, s["x"][a:b]) for a, b in cuts(len(s["x"]))]
    jobs += [pool.submit(oracle.dot, s["dx"][a:b], s["dy"][a:b]) for a, b in cuts(len(s["dx"]))]
    m = s["A"].shape[0]
    rows = max(1, -(-m // k))
    jobs += [pool.submit(oracle.gemv, s["A"][a:a + rows], s["gx"], s["gy"][a:a + rows], ALPHA, BETA)
             for a in range(0, m, rows)]
    for j in jobs:
        j.result()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(budget_s: float = 10.0, frac_shift: int = 3, cores_budget_s: float = 5.0):
    """The oracle as it stands, single-threaded, on a bounded sample (rank 0, N=1); plus the
    same oracle run over all host cores under "all_cores"."""
    from concurrent.futures import ThreadPoolExecutor
    s = oracle_sample(frac_shift)
    oracle_step(s)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle_step(s)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    out = {"value": round(s["bytes"] * reps / dt / 1e9, 3), "unit": "GB/s", "cores": 1,
           "kind": "oracle",
           "sample": f"{reps} x ({s['desc']}) in {dt:.1f} s, fp64 Neumaier C oracle, 1 thread"}
    k = len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(k) as pool:
        oracle_step_cores(s, pool, k)  # warm
        reps, t0 = 0, time.perf_counter()
        while True:
            oracle_step_cores(s, pool, k)
            reps += 1
            if time.perf_counter() - t0 >= cores_budget_s:
                break
        dt = time.perf_counter() - t0
    out["host_cpu"] = _cpu_model()
    out["all_cores"] = {"value": round(s["bytes"] * reps / dt / 1e9, 3), "unit": "GB/s",
                        "cores": k, "sample": f"{reps} x (same step, every operand in {k} "
                        f"shards on {k} threads) in {dt:.1f} s"}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # under torchrun only rank 0 runs the CPU oracle
    frac_shift = 4
    s = oracle_sample(frac_shift)
    for _ in range(args.warmup):
        oracle_step(s)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(s)
    dt = time.perf_counter() - t0
    val = s["bytes"] * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": "achieved HBM GB/s (fraction of 8 TB/s) for "
        "asum/dot/scal/gemv at 1/2/4/8 B200", "value": round(val, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "scal+asum 2^28, dot 2^26, gemv 8192x8192 (sampled 1/16)",
                   "global_batch": 1, "parallelism": "cpu-1thread"},
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": s["desc"]},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- lift arm
def _dbg(msg):
    if os.environ.get("LIFT_BENCH_DEBUG"):
        print(f"[rank {os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def run_lift(args):
    import torch
    import torch.distributed as dist

    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    from paper_1502_02389_b200 import dist as ldist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # LIFT_DIST_BACKEND=gloo (test only) runs N ranks on fewer GPUs: exercises the N>1
    # code path on a single-GPU box; the performance numbers of such a run are meaningless.
    backend = os.environ.get("LIFT_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    group = None
    stream = torch.cuda.current_stream(dev)

    # ---- inputs, resident in HBM (rank r owns global slice r: weak scaling) ----------
    def fill(n, tid, i0, lo, hi):
        t = torch.empty(n, dtype=torch.float32, device=dev)
        return gen.fill_device(t, 0, tid, i0, gen.DIST_UNIFORM, lo, hi)

    x_v = fill(N_VEC, gen.TID_X, rank * N_VEC, -1.0, 1.0)
    y_v = torch.empty(N_VEC, dtype=torch.float32, device=dev)
    x_d = fill(N_DOT, gen.TID_X, rank * N_DOT, 0.0, 1.0)
    y_d = fill(N_DOT, gen.TID_Y, rank * N_DOT, 0.0, 2.0)
    A = fill(GEMV_M * GEMV_N, gen.TID_A, rank * GEMV_M * GEMV_N, 0.0, 3.0).view(GEMV_M, GEMV_N)
    g_x = fill(GEMV_N, gen.TID_X, 0, 0.0, 1.0)  # replicated
    g_y = fill(GEMV_M, gen.TID_Y, rank * GEMV_M, 0.0, 2.0)
    g_out = torch.empty(GEMV_M, dtype=torch.float32, device=dev)
    g_full = torch.empty(GEMV_M * world, dtype=torch.float32, device=dev)
    r_asum = torch.empty(1, dtype=torch.float32, device=dev)
    r_dot = torch.empty(1, dtype=torch.float32, device=dev)
    ws_a = lift.Workspace(N_VEC, dev)
    ws_d = lift.Workspace(N_DOT, dev)
    # X1 for asum/dot at N > 1: the combine fused into the reduction kernel (NEXT-1,
    # peer-memory exchange); LIFT_X1=nccl selects all-gather + lift_combine instead.
    x1_mode = os.environ.get("LIFT_X1", "fused") if world > 1 else "none"
    xchg, x1_note = None, ""
    if x1_mode == "fused":
        xchg, x1_note = fused_exchange_or_none(lift, ldist, torch, dist, group, dev)
        if xchg is None:  # every rank falls back together (agreed below): the NCCL X1 path
            x1_mode = "nccl"

    def x_asum(x, out, ws):
        return xchg.asum(x, out=out, ws=ws) if xchg else ldist.sharded_asum(x, group, out=out, ws=ws)

    def x_dot(x, y, out, ws):
        return (xchg.dot(x, y, out=out, ws=ws) if xchg
                else ldist.sharded_dot(x, y, group, out=out, ws=ws))

    def x_gemv(A, gx, gy, out_full, out_slice):
        if xchg:  # rows land in every rank's full y inside the gemv kernel
            return xchg.gemv(A, gx, gy, ALPHA, BETA, GEMV_M * world, rank * GEMV_M)
        return ldist.sharded_gemv(A, gx, gy, ALPHA, BETA, GEMV_M * world, group,
                                  out_full=out_full, out_slice=out_slice)
    torch.cuda.synchronize()

    def op_scal():
        lift.scal(ALPHA_SCAL, x_v, out=y_v)

    def op_asum():
        if world == 1:
            lift.asum(x_v, out=r_asum, ws=ws_a)
        else:
            x_asum(x_v, r_asum, ws_a)

    def op_dot():
        if world == 1:
            lift.dot(x_d, y_d, out=r_dot, ws=ws_d)
        else:
            x_dot(x_d, y_d, r_dot, ws_d)

    def op_gemv():
        if world == 1:
            lift.gemv(A, g_x, g_y, ALPHA, BETA, out=g_out)
        else:
            x_gemv(A, g_x, g_y, g_full, g_out)

    op_fn = {"scal": op_scal, "asum": op_asum, "dot": op_dot, "gemv": op_gemv}

    def step(ev=None):
        """One pass of the hot path (in OPS order); ev = per-op event boundaries or None."""
        for i, op in enumerate(OPS):
            if ev is not None:
                ev[i].record(stream)
            op_fn[op]()
        if ev is not None:
            ev[len(OPS)].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    _dbg("inputs ready")
    for _ in range(max(args.warmup, 0)):
        step()
    barrier()
    _dbg("warm-up done")

    # ---- timed region A (the headline): K steps, events only at its two ends ----------
    # Events recorded BETWEEN kernels break the programmatic-dependent-launch overlap of
    # consecutive kernels (measured: 606.6 vs 588.2 us per step, scripts/step_ab.py), so
    # the headline region has none; per-op times come from region B.
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    barrier()
    t_wall0 = time.time()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        step()
    end.record(stream)
    barrier()
    t_wall1 = time.time()
    # ---- timed region B (instrumented): the same K steps with per-op events on the
    # launching stream -> per-op durations (roofline.achieved), shares, per-step spread
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(OPS) + 1)]
           for _ in range(args.steps)]
    barrier()
    startb = torch.cuda.Event(enable_timing=True)
    endb = torch.cuda.Event(enable_timing=True)
    startb.record(stream)
    for k in range(args.steps):
        step(evs[k])
    endb.record(stream)
    barrier()
    # keep the GPU busy until the sampler has seen the load (short K on a fast GPU).
    # Untimed and rank-local: only the kernels, never the X1 collectives (rank 0 alone
    # runs this loop, so a collective here would deadlock the other ranks).
    while sampler and len([1 for (t, _) in sampler.rows if t >= t_wall0]) < 5 \
            and time.time() - t_wall0 < 10:
        lift.scal(ALPHA_SCAL, x_v, out=y_v)
        lift.asum(x_v, out=r_asum, ws=ws_a)
        lift.dot(x_d, y_d, out=r_dot, ws=ws_d)
        lift.gemv(A, g_x, g_y, ALPHA, BETA, out=g_out)
        torch.cuda.synchronize()
    t_wall2 = time.time()
    if sampler:
        sampler.stop()
    _dbg("timed regions done")
    total_ms = max_over_ranks(start.elapsed_time(end))
    total_b_ms = max_over_ranks(startb.elapsed_time(endb))
    per_op_ms = {op: 0.0 for op in OPS}
    step_ms_b = []
    for k in range(args.steps):
        for i, op in enumerate(OPS):
            per_op_ms[op] += evs[k][i].elapsed_time(evs[k][i + 1])
        step_ms_b.append(evs[k][0].elapsed_time(evs[k][len(OPS)]))
    per_op_ms = {op: max_over_ranks(v) / args.steps for op, v in per_op_ms.items()}
    step_ms_b.sort()

    def pct(q):
        return step_ms_b[min(len(step_ms_b) - 1, int(q * (len(step_ms_b) - 1) + 0.5))]

    ob = op_bytes(world)
    oe = op_elems()
    step_bytes = sum(ob.values())
    ms_per_step = total_ms / args.steps
    value = step_bytes * world / (ms_per_step * 1e-3) / 1e9  # whole-job GB/s

    # ---- e2e: the same step through the public API with pinned HOST buffers --------
    e2e = None
    _dbg("per-op times reduced")
    if not args.no_e2e:
        e2e = run_e2e(args, lift, ldist, gen, torch, dist, world, rank, dev, group, stream,
                      max_over_ranks, barrier, step_bytes, x_asum, x_dot, x_gemv)

    peak, peak_src = load_peaks()
    traffic = load_traffic()
    dom = max(OPS, key=lambda o: per_op_ms[o])
    dom_gbs = ob[dom] / (per_op_ms[dom] * 1e-3) / 1e9
    ms_b = total_b_ms / args.steps
    per_op = {op: {"ms": round(per_op_ms[op], 4), "bytes": ob[op], "elements": oe[op],
                   "GB/s": round(ob[op] / (per_op_ms[op] * 1e-3) / 1e9, 1),
                   "elements_per_s": float(f"{oe[op] / (per_op_ms[op] * 1e-3):.4g}"),
                   "frac_measured_peak": round(ob[op] / (per_op_ms[op] * 1e-3) / 1e9 / peak, 4),
                   "frac_8TBs": round(ob[op] / (per_op_ms[op] * 1e-3) / 1e9 / NOMINAL_HBM, 4),
                   "share_of_step": round(per_op_ms[op] / ms_b, 4)}
              for op in OPS}
    scaling = None
    if world > 1 and not args.no_extras:
        scaling = scaling_configs(args, lift, ldist, gen, torch, dist, world, rank, dev, group,
                                  max_over_ranks, barrier, x1_mode, xchg)

    if rank == 0:
        launches_per_step = 4 + (2 if x1_mode == "nccl" else 0)
        line = {
            "metric": "achieved HBM GB/s (fraction of 8 TB/s) for asum/dot/scal/gemv at "
                      "1/2/4/8 B200",
            "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "elements_per_s": float(f"{sum(oe.values()) * world / (ms_per_step * 1e-3):.4g}"),
            "frac_of_8TBs": round(value / world / NOMINAL_HBM, 4),
            "timing": {"headline": "region A: K steps between two CUDA events (no events "
                                   "between kernels)",
                       "instrumented_ms_per_step": round(ms_b, 4),
                       "instrumented_step_ms": {"median": round(pct(0.5), 4),
                                                "p10": round(pct(0.1), 4),
                                                "p90": round(pct(0.9), 4)},
                       "per_op_from": "region B: the same K steps with an event before and "
                                      "after every kernel on the launching stream"},
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "accum": "asum f32 4-term runs then f64; dot/gemv exact products in f64",
            "data": "synthetic (seeded counter-based generator, device-filled)",
            "config": {"workload": "step = scal+asum fp32 n=2^28 (configs[2]) + dot fp32 "
                                   "n=2^26 (configs[1]) + gemv 8192x8192 a=1.5 b=0.5 "
                                   "(configs[3]), per rank",
                       "global_batch": world, "parallelism": f"shard{world} (weak)",
                       "x1": {"none": "single GPU", "fused": "asum/dot combine and the gemv y "
                              "all-gather fused into the kernels over peer memory (no NCCL "
                              "launch in the step)",
                              "nccl": "all-gather + lift_combine; gemv y all-gather"}[x1_mode]
                             + (f" [{x1_note}]" if x1_note else ""),
                       "l2": "no flush: every operand >= 256 MiB > 126 MB L2",
                       "frac_of_8TBs": round(value / world / NOMINAL_HBM, 4)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(dom_gbs, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(dom_gbs / peak, 4),
                         "traffic": traffic.get(dom), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": ob[dom]},
            "per_op": per_op,
            "gpu_launches": launches_per_step * args.steps,
            "scaling_configs": scaling,
            "clocks": sampler.summary(t_wall0, max(t_wall1, t_wall2)) if sampler else None,
            "e2e": e2e,
        }
        if not args.no_extras:
            line["next_rows"] = next_rows(lift, gen, torch, dev, stream, x_v, y_v, r_asum, ws_a)
            if world == 1:
                line["baseline_configs"] = baseline_configs(lift, gen, torch, dev, x_v, y_v, x_d, y_d,
                                                            A, g_x, g_y, g_out)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_budget)
        print(json.dumps(line), flush=True)
    if xchg is not None:
        xchg.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def fused_exchange_or_none(lift, ldist, torch, dist, group, dev):
    """The NEXT-1 peer-memory exchange, probed end to end once (a fused asum over one chunk
    per rank, its error word checked); all ranks agree (all-reduce MIN) so that a node where
    CUDA IPC / P2P does not work falls back to the NCCL X1 path on every rank instead of
    failing the run.  Returns (PeerExchange or None, note)."""
    ex, note = None, ""
    try:
        ex = ldist.PeerExchange(group, device=dev)
        if os.environ.get("LIFT_X1_PROBE_FAIL") == str(dist.get_rank(group)):
            raise RuntimeError("LIFT_X1_PROBE_FAIL test hook")  # exercises the fallback
        probe = torch.ones(lift.CHUNK_ELEMS, dtype=torch.float32, device=dev)
        r = ex.asum(probe)
        torch.cuda.synchronize(dev)
        ex.check()
        if float(r.item()) != float(lift.CHUNK_ELEMS * dist.get_world_size(group)):
            raise RuntimeError(f"probe asum {float(r.item())}")
    except Exception as e:  # noqa: BLE001 — any failure selects the NCCL path
        note = f"fused exchange unavailable ({type(e).__name__}: {str(e)[:160]}); NCCL X1 path"
        ex = None
    ok = torch.tensor([1 if ex is not None else 0], dtype=torch.int32,
                      device=dev if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) == 0 and ex is not None:
        ex.close()
        ex = None
        note = note or "fused exchange unavailable on another rank; NCCL X1 path"
    return ex, note


def scaling_configs(args, lift, ldist, gen, torch, dist, world, rank, dev, group,
                    max_over_ranks, barrier, x1_mode, xchg):
    """BASELINE.json configs[3] and [4] as STRONG scaling (the global problem is fixed):
      C4  gemv 8192 x 8192, alpha=1.5 beta=0.5: rank r owns rows row_range(8192, r, N)
      C5  dot n = 2^31: rank r owns shard_range(2^31, r, N) (canonical-group aligned)
    Per config: 'kernel' = the rank's local launch only; 'fused' = end to end through the
    NEXT-1 path (exchange inside the kernel over IPC-mapped peer memory); 'nccl' = local
    kernel + torch.distributed all-gather + lift_combine (C5) / y all-gather (C4).  Each
    time: `reps` back-to-back calls between two events, median of 5, max over ranks.
    efficiency = t(1) / (N * t(N)), t(1) measured in this run on rank 0's GPU (unsharded).
    Every rank checks that both X1 paths give the unsharded bits."""
    reps = 10
    M = N = GEMV_M
    NC5 = 1 << 31

    def timed(fn, collective=True, nreps=reps):
        ts = []
        for _ in range(5):
            if collective:
                barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(nreps):
                fn()
            e.record()
            e.synchronize()
            t = s.elapsed_time(e) / nreps
            ts.append(max_over_ranks(t) if collective else t)
        return sorted(ts)[2]

    def fill(n, tid, i0, lo, hi):
        return gen.fill_device(torch.empty(n, dtype=torch.float32, device=dev), 0, tid, i0,
                               gen.DIST_UNIFORM, lo, hi)

    ex, ex_note = (xchg, "") if xchg is not None else fused_exchange_or_none(
        lift, ldist, torch, dist, group, dev)
    out = {"note": "strong scaling: fixed global problem split over N ranks; kernel = local "
                   "launch only, fused / nccl = end to end including the X1 exchange; "
                   "median of 5 x %d calls, max over ranks" % reps}

    # ---- C4: gemv rows ---------------------------------------------------------------
    r0, r1 = ldist.row_range(M, rank, world)
    A = fill((r1 - r0) * N, gen.TID_A, r0 * N, 0.0, 3.0).view(r1 - r0, N)
    gx = fill(N, gen.TID_X, 0, 0.0, 1.0)
    gy = fill(r1 - r0, gen.TID_Y, r0, 0.0, 2.0)
    go = torch.empty(r1 - r0, device=dev)
    gfull = torch.empty(M, device=dev)
    t_k = timed(lambda: lift.gemv(A, gx, gy, ALPHA, BETA, out=go))
    t_f = timed(lambda: ex.gemv(A, gx, gy, ALPHA, BETA, M, r0)) if ex else None
    yf = ex.gemv(A, gx, gy, ALPHA, BETA, M, r0).clone() if ex else None
    t_n = timed(lambda: ldist.sharded_gemv(A, gx, gy, ALPHA, BETA, M, group, out_full=gfull,
                                           out_slice=go))
    yn = ldist.sharded_gemv(A, gx, gy, ALPHA, BETA, M, group, out_full=gfull, out_slice=go).clone()
    ref = {}
    if rank == 0:  # the unsharded problem on this GPU: t(1) and the reference bits
        Af = fill(M * N, gen.TID_A, 0, 0.0, 3.0).view(M, N)
        gyf = fill(M, gen.TID_Y, 0, 0.0, 2.0)
        gof = torch.empty(M, device=dev)
        ref["t1"] = timed(lambda: lift.gemv(Af, gx, gyf, ALPHA, BETA, out=gof), collective=False)
        ref["bits"] = lift.gemv(Af, gx, gyf, ALPHA, BETA, out=gof).clone()
        del Af
    barrier()
    bytes_all = 4 * (M * N + world * N + 2 * M)
    c4 = {"rows_per_rank": r1 - r0}
    paths = ("kernel", "fused", "nccl") if ex else ("kernel", "nccl")
    if not ex:
        c4["fused"] = {"unavailable": ex_note}
    for k, t in (("kernel", t_k), ("fused", t_f), ("nccl", t_n)):
        if t is None:
            continue
        c4[k] = {"ms": round(t, 4), "GB/s": round(bytes_all / (t * 1e-3) / 1e9, 1),
                 "elements_per_s": float(f"{M * N / (t * 1e-3):.4g}"),
                 "frac_of_8TBs_per_gpu": round(bytes_all / (t * 1e-3) / 1e9 / world / NOMINAL_HBM, 4)}
    if rank == 0:
        c4["t1_ms"] = round(ref["t1"], 4)
        for k in paths:
            c4[k]["efficiency_vs_1"] = round(ref["t1"] / (world * c4[k]["ms"]), 4)
        c4["bits_equal_unsharded"] = bool(
            (yf is None or torch.equal(yf.view(torch.int32), ref["bits"].view(torch.int32)))
            and torch.equal(yn.view(torch.int32), ref["bits"].view(torch.int32)))
    out["C4 gemv 8192x8192 row-sharded"] = c4
    del A

    # ---- C5: dot over 2^31 -----------------------------------------------------------
    a0, a1 = ldist.shard_range(NC5, rank, world)
    x = fill(a1 - a0, gen.TID_X, a0, 0.0, 1.0)
    y = fill(a1 - a0, gen.TID_Y, a0, 0.0, 2.0)
    ws = lift.Workspace(a1 - a0, dev)
    r = torch.empty(1, device=dev)
    p64 = torch.empty(1, dtype=torch.float64, device=dev)
    t_k = timed(lambda: lift.dot_partial(x, y, out=p64, ws=ws), nreps=3)
    t_f = timed(lambda: ex.dot(x, y, out=r, ws=ws), nreps=3) if ex else None
    rf = ex.dot(x, y, out=torch.empty(1, device=dev), ws=ws) if ex else None
    t_n = timed(lambda: ldist.sharded_dot(x, y, group, out=r, ws=ws), nreps=3)
    rn = ldist.sharded_dot(x, y, group, out=torch.empty(1, device=dev), ws=ws)
    del x, y
    if rank == 0:
        xf = fill(NC5, gen.TID_X, 0, 0.0, 1.0)
        yf5 = fill(NC5, gen.TID_Y, 0, 0.0, 2.0)
        wsf = lift.Workspace(NC5, dev)
        ref["t1"] = timed(lambda: lift.dot(xf, yf5, out=r, ws=wsf), collective=False, nreps=3)
        ref["bits"] = lift.dot(xf, yf5, out=torch.empty(1, device=dev), ws=wsf)
        del xf, yf5, wsf
    barrier()
    c5 = {"elements_per_rank": a1 - a0}
    if not ex:
        c5["fused"] = {"unavailable": ex_note}
    for k, t in (("kernel", t_k), ("fused", t_f), ("nccl", t_n)):
        if t is None:
            continue
        c5[k] = {"ms": round(t, 4), "GB/s": round(8 * NC5 / (t * 1e-3) / 1e9, 1),
                 "elements_per_s": float(f"{NC5 / (t * 1e-3):.4g}"),
                 "frac_of_8TBs_per_gpu": round(8 * NC5 / (t * 1e-3) / 1e9 / world / NOMINAL_HBM, 4)}
    if rank == 0:
        c5["t1_ms"] = round(ref["t1"], 4)
        for k in paths:
            c5[k]["efficiency_vs_1"] = round(ref["t1"] / (world * c5[k]["ms"]), 4)
        c5["bits_equal_unsharded"] = bool(
            (rf is None or torch.equal(rf.view(torch.int32), ref["bits"].view(torch.int32)))
            and torch.equal(rn.view(torch.int32), ref["bits"].view(torch.int32)))
    out["C5 dot 2^31 sharded"] = c5
    if xchg is None and ex is not None:
        ex.close()
    torch.cuda.empty_cache()
    return out


def baseline_configs(lift, gen, torch, dev, x_v, y_v, x_d, y_d, A, g_x, g_y, g_out, reps=20):
    """BASELINE.json's configs C1-C5 on this GPU, each alone: `reps` back-to-back launches in
    one CUDA graph (median of 5 replays), reusing the step's operands where they match.
    Operands >= 256 MiB exceed the 126 MB L2; C1 (4 MiB) is L2-resident by nature."""
    cs = torch.cuda.Stream(device=dev)

    def timed(fn, nbytes, n_reps=reps):
        torch.cuda.synchronize()
        with torch.cuda.stream(cs):
            fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for _ in range(n_reps):
                    fn()
            ts = []
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(cs)
                g.replay()
                e.record(cs)
                e.synchronize()
                ts.append(s.elapsed_time(e) / n_reps * 1e3)
        us = sorted(ts)[2]
        gbs = nbytes / (us * 1e-6) / 1e9
        return {"us": round(us, 2), "GB/s": round(gbs, 1), "frac_8TBs": round(gbs / NOMINAL_HBM, 3)}

    r = torch.empty(1, dtype=torch.float32, device=dev)
    ws = lift.Workspace(1 << 28, dev)
    out = {"note": "each config alone, CUDA-graph back-to-back launches, median of 5"}
    out["C1 asum 2^20 (L2-resident)"] = timed(lambda: lift.asum(x_v[:1 << 20], out=r, ws=ws), 4 << 20)
    # C2: 2^24 rotates over 4 disjoint slices of the step's operands (so it streams HBM)
    k = [0]

    def dot24():
        i = k[0] % 4
        k[0] += 1
        lift.dot(x_v[i << 24:(i + 1) << 24], y_v[i << 24:(i + 1) << 24], out=r, ws=ws)
    y_v.copy_(x_v)
    out["C2 dot 2^24"] = timed(dot24, 8 << 24)
    out["C2 dot 2^26"] = timed(lambda: lift.dot(x_d, y_d, out=r, ws=ws), 8 << 26)
    out["C3 scal 2^28"] = timed(lambda: lift.scal(ALPHA_SCAL, x_v, out=y_v), 8 << 28)
    out["C3 asum 2^28"] = timed(lambda: lift.asum(x_v, out=r, ws=ws), 4 << 28)
    m, n = A.shape
    # C4: rotates over 3 copies of A (> 2x L2), like C2 2^24 over disjoint slices, so every
    # launch streams its matrix from HBM (scripts/ab.py / tune.py measure the same way)
    As = [A] + [A.clone() for _ in range(2)]
    k4 = [0]

    def gemv_rot():
        i = k4[0] % len(As)
        k4[0] += 1
        lift.gemv(As[i], g_x, g_y, ALPHA, BETA, out=g_out)
    out["C4 gemv 8192x8192 (p=1)"] = timed(gemv_rot, 4 * (m * n + n + 2 * m))
    del As
    sh = m // 8
    ks = [0]

    def shard_rot():  # the 8 disjoint p=8 row blocks in turn (268 MB > L2): from HBM
        i = ks[0] % 8
        ks[0] += 1
        lift.gemv(A[i * sh:(i + 1) * sh], g_x, g_y[:sh], ALPHA, BETA, out=g_out[:sh])
    out["C4 gemv 1024x8192 (one p=8 shard, from HBM)"] = timed(shard_rot, 4 * (sh * n + n + 2 * sh))
    out["C4 gemv 1024x8192 (one p=8 shard, L2-warm)"] = timed(
        lambda: lift.gemv(A[:sh], g_x, g_y[:sh], ALPHA, BETA, out=g_out[:sh]), 4 * (sh * n + n + 2 * sh))
    # C5: dot over 2^31 elements (16 GiB of inputs) on this one GPU, if memory allows
    free, _ = torch.cuda.mem_get_info(dev)
    if free > (20 << 30):
        bx = gen.fill_device(torch.empty(1 << 31, dtype=torch.float32, device=dev), 0, gen.TID_X, 0,
                             gen.DIST_UNIFORM, 0.0, 1.0)
        by = gen.fill_device(torch.empty(1 << 31, dtype=torch.float32, device=dev), 0, gen.TID_Y, 0,
                             gen.DIST_UNIFORM, 0.0, 2.0)
        wsb = lift.Workspace(1 << 31, dev)
        out["C5 dot 2^31 (p=1)"] = timed(lambda: lift.dot(bx, by, out=r, ws=wsb), 8 << 31, n_reps=5)
        del bx, by, wsb
    return out


def next_rows(lift, gen, torch, dev, stream, x_v, y_v, r, ws, reps=20):
    """NEXT rows measured beside the step (not part of it): the fused scal+asum (NEXT-2)
    on the step's x, and BlackScholes on the paper's 4M prices (NEXT-3).  Each is
    `reps` launches captured in one CUDA graph (a 7 us kernel launched from Python would
    measure the launch path), median of 5 replays."""
    cs = torch.cuda.Stream(device=dev)  # graphs are captured on a side stream

    def timed(fns):
        for f in fns[:3]:
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for i in range(reps):
                fns[i % len(fns)]()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(cs)
            g.replay()
            e.record(cs)
            e.synchronize()
            ts.append(s.elapsed_time(e) / reps * 1e3)  # us
        return sorted(ts)[2]
    n = x_v.numel()
    torch.cuda.synchronize()
    with torch.cuda.stream(cs):
        us_f = timed([lambda: lift.scal_asum(ALPHA_SCAL, x_v, out=y_v, result=r, ws=ws)])
        # 4 rotating price/call/put sets (4 x 48 MB > 126 MB L2), so the launches stream HBM
        nb = 4 * 1024 * 1024
        sets = []
        for c in range(4):
            sp = gen.fill_device(torch.empty(nb, dtype=torch.float32, device=dev), c, gen.TID_X, 0,
                                 gen.DIST_UNIFORM, 10.0, 200.0)
            sets.append((sp, torch.empty_like(sp), torch.empty_like(sp)))
        us_b = timed([lambda t=t: lift.blackscholes(t[0], 100.0, 0.05, 0.2, 1.0, call=t[1], put=t[2])
                      for t in sets])
    return {
        "scal_asum_fused": {"n": n, "us": round(us_f, 2), "GB/s": round(8 * n / us_f / 1e3, 1),
                            "vs_separate_scal_then_asum_bytes": "8 vs 12 B/element"},
        "blackscholes": {"n": nb, "us": round(us_b, 2), "Goptions/s": round(nb / us_b / 1e3, 2),
                         "GB/s": round(12 * nb / us_b / 1e3, 1),
                         "bound": "memory (12 B/price; 4 rotating 48 MB sets > L2, graph replay)"},
    }


def run_e2e(args, lift, ldist, gen, torch, dist, world, rank, dev, group, stream,
            max_over_ranks, barrier, step_bytes, x_asum, x_dot, x_gemv):
    """Same metric, end to end: every step copies its inputs from pinned host memory,
    runs the step through the public API and reads every result back to the host."""
    steps = max(1, min(args.steps, args.e2e_steps))

    def host(n, tid, i0, lo, hi):
        t = torch.empty(n, dtype=torch.float32).pin_memory()
        gen.fill_host(t.numpy(), 0, tid, i0, gen.DIST_UNIFORM, lo, hi)
        return t

    h_x = host(N_VEC, gen.TID_X, rank * N_VEC, -1.0, 1.0)
    h_dx = host(N_DOT, gen.TID_X, rank * N_DOT, 0.0, 1.0)
    h_dy = host(N_DOT, gen.TID_Y, rank * N_DOT, 0.0, 2.0)
    h_A = host(GEMV_M * GEMV_N, gen.TID_A, rank * GEMV_M * GEMV_N, 0.0, 3.0)
    h_gx = host(GEMV_N, gen.TID_X, 0, 0.0, 1.0)
    h_gy = host(GEMV_M, gen.TID_Y, rank * GEMV_M, 0.0, 2.0)
    h_yv = torch.empty(N_VEC, dtype=torch.float32).pin_memory()
    h_res = torch.empty(2, dtype=torch.float32).pin_memory()
    h_g = torch.empty(GEMV_M * world, dtype=torch.float32).pin_memory()
    d = {k: torch.empty(v.numel(), dtype=torch.float32, device=dev)
         for k, v in (("x", h_x), ("dx", h_dx), ("dy", h_dy), ("A", h_A), ("gx", h_gx),
                      ("gy", h_gy))}
    d_yv = torch.empty(N_VEC, dtype=torch.float32, device=dev)
    d_res = torch.empty(2, dtype=torch.float32, device=dev)
    d_g = torch.empty(GEMV_M, dtype=torch.float32, device=dev)
    d_gf = torch.empty(GEMV_M * world, dtype=torch.float32, device=dev)
    ws_a, ws_d = lift.Workspace(N_VEC, dev), lift.Workspace(N_DOT, dev)
    h2d = sum(v.numel() * 4 for v in (h_x, h_dx, h_dy, h_A, h_gx, h_gy))
    d2h = (N_VEC + 2 + GEMV_M * world) * 4

    # Pipelined over three streams (copy engines H2D and D2H run concurrently with the
    # kernels): x arrives in NCH chunks and scal runs chunk by chunk as they land (its
    # output streams back while later chunks arrive); asum, dot and gemv start as soon
    # as their inputs are resident.  Every byte of every input still crosses PCIe each
    # step, and every result comes back.
    NCH = 8
    cs = N_VEC // NCH
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s_cmp = stream
    ev = lambda: torch.cuda.Event()  # noqa: E731
    prev_done = [None]  # event: previous step fully finished (all three streams)

    def e2e_step():
        ev_x = [ev() for _ in range(NCH)]
        ev_y = [ev() for _ in range(NCH)]
        ev_dot, ev_g, ev_res, ev_out = ev(), ev(), ev(), ev()
        with torch.cuda.stream(s_h2d):
            if prev_done[0] is not None:
                s_h2d.wait_event(prev_done[0])  # buffers are reused across steps
            for i in range(NCH):
                d["x"][i * cs:(i + 1) * cs].copy_(h_x[i * cs:(i + 1) * cs], non_blocking=True)
                ev_x[i].record(s_h2d)
            d["dx"].copy_(h_dx, non_blocking=True)
            d["dy"].copy_(h_dy, non_blocking=True)
            ev_dot.record(s_h2d)
            for k, h in (("A", h_A), ("gx", h_gx), ("gy", h_gy)):
                d[k].copy_(h, non_blocking=True)
            ev_g.record(s_h2d)
        with torch.cuda.stream(s_cmp):
            for i in range(NCH):
                s_cmp.wait_event(ev_x[i])
                lift.scal(ALPHA_SCAL, d["x"][i * cs:(i + 1) * cs], out=d_yv[i * cs:(i + 1) * cs])
                ev_y[i].record(s_cmp)
            A = d["A"].view(GEMV_M, GEMV_N)
            if world == 1:
                lift.asum(d["x"], out=d_res[0:1], ws=ws_a)
                s_cmp.wait_event(ev_dot)
                lift.dot(d["dx"], d["dy"], out=d_res[1:2], ws=ws_d)
                s_cmp.wait_event(ev_g)
                lift.gemv(A, d["gx"], d["gy"], ALPHA, BETA, out=d_gf)
            else:
                x_asum(d["x"], d_res[0:1], ws_a)
                s_cmp.wait_event(ev_dot)
                x_dot(d["dx"], d["dy"], d_res[1:2], ws_d)
                s_cmp.wait_event(ev_g)
                yf = x_gemv(A, d["gx"], d["gy"], d_gf, d_g)
                if yf.data_ptr() != d_gf.data_ptr():
                    d_gf.copy_(yf)
            ev_res.record(s_cmp)
        with torch.cuda.stream(s_d2h):
            for i in range(NCH):
                s_d2h.wait_event(ev_y[i])
                h_yv[i * cs:(i + 1) * cs].copy_(d_yv[i * cs:(i + 1) * cs], non_blocking=True)
            s_d2h.wait_event(ev_res)
            h_res.copy_(d_res, non_blocking=True)
            h_g.copy_(d_gf, non_blocking=True)
            ev_out.record(s_d2h)
        prev_done[0] = ev_out

    barrier()  # ranks enter the first exchange together (host buffer filling can skew them)
    e2e_step()
    torch.cuda.synchronize()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    s_h2d.wait_event(s)
    s_d2h.wait_event(s)
    prev_done[0] = s
    for _ in range(steps):
        e2e_step()
    stream.wait_event(prev_done[0])
    e.record(stream)
    barrier()
    ms = max_over_ranks(s.elapsed_time(e)) / steps
    return {"value": round(step_bytes * world / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3),
            "steps": steps, "pipeline": f"3 streams (H2D / kernels / D2H), x in {NCH} chunks",
            "launches_per_step": NCH + 3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="lift", choices=["lift", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT-row timings")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "lift":
        print("note: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_lift(args)


if __name__ == "__main__":
    sys.exit(main())
