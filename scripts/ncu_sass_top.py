"""Top SASS instructions by warp-stall samples from an ncu report (--import-source, -lineinfo):
    python scripts/ncu_sass_top.py report.ncu-rep [N] [--all] [--kernel REGEX]
--all prints every instruction in address order with its samples (for reading the loop);
--kernel picks the kernel of a multi-kernel report (ncu -k regex:REGEX)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
kf = []
if "--kernel" in sys.argv:
    kf = ["-k", "regex:" + sys.argv[sys.argv.index("--kernel") + 1]]
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
nxt = [i for i, l in enumerate(lines) if i > 0 and l.startswith('"Kernel Name"')]
if nxt:  # the page may list a kernel more than once: keep the first block
    lines = lines[:nxt[0]]
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
data = [(r[ia], r[isrc].strip(), int(r[iss] or 0), r[iex]) for r in rows[1:] if len(r) == len(h)]
tot = sum(d[2] for d in data)
print(f"# {lines[0][:120]}\n# total samples {tot}")
if "--all" in sys.argv:
    for a, s, n, e in data:
        print(f"{a[-5:]} {n:6d} {e:>9s}  {s}")
else:
    for a, s, n, e in sorted(data, key=lambda d: -d[2])[:N]:
        print(f"{n:6d} {100 * n / max(tot, 1):5.1f}%  {a[-5:]}  {s}")
