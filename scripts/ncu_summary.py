"""Summarise an ncu --set full report (.ncu-rep) into a small text table.

    python scripts/ncu_summary.py gpurun_out/prof_r1.ncu-rep > profiles/...txt
Also writes per-kernel dram bytes per launch to profiles/traffic.json when --traffic is
given (bench.py reads it for roofline.traffic)."""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_thru_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_sm_%"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall_long_sb"),
    ("smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "stall_long_sb_%"),
    ("smsp__warp_issue_stalled_barrier_per_warp_active.pct", "stall_barrier_%"),
    ("smsp__warp_issue_stalled_membar_per_warp_active.pct", "stall_membar_%"),
    ("smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "stall_lg_throttle_%"),
    ("smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct", "stall_math_thr_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    traffic = {}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[idx["Kernel Name"]]
        short = re.sub(r"void lift::|\(.*", "", name)[:60]
        print(f"== {short}")
        for k, lab in KEYS:
            if k in idx:
                print(f"   {lab:22s} {r[idx[k]]:>16s} {units[idx[k]]}")
        try:
            rd = float(r[idx["dram__bytes_read.sum"]].replace(",", ""))
            wr = float(r[idx["dram__bytes_write.sum"]].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            u1 = mult.get(units[idx["dram__bytes_read.sum"]], 1)
            u2 = mult.get(units[idx["dram__bytes_write.sum"]], 1)
            op = ("scal" if "scal" in short else "gemv" if "gemv" in short else
                  "dot" if "DotOp" in name else "asum" if "AsumOp" in name else short)
            traffic[op] = int(rd * u1 + wr * u2)
        except Exception:
            pass
    if "--traffic" in sys.argv:
        with open(sys.argv[sys.argv.index("--traffic") + 1], "w") as f:
            json.dump(traffic, f, indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
