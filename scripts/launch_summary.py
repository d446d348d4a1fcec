"""Summarise an ncu --metrics launch list (csv) per op: launches, mean us, share, dram MB."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[h.index("Kernel Name")]
    short = ("scal" if "scal" in name else "gemv" if "gemv" in name else "dot" if "DotOp" in name
             else "asum" if "AsumOp" in name else "combine" if "combine" in name else name[:30])
    m = r[h.index("Metric Name")]
    v = float(r[h.index("Metric Value")].replace(",", ""))
    agg.setdefault(short, collections.defaultdict(list))[m].append(v)
tot = sum(sum(d["gpu__time_duration.sum"]) for d in agg.values())
print(f"# ncu launch list: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# cold-cache, serialised per-launch times (ncu): compare SHARES with bench.py per_op")
print("op       launches   mean_us   share   dram_read_MB  dram_write_MB")
for k, d in agg.items():
    t = d["gpu__time_duration.sum"]
    print(f"{k:8s} {len(t):8d} {sum(t) / len(t) / 1e3:9.2f} {sum(t) / tot:7.3f} "
          f"{sum(d['dram__bytes_read.sum']) / len(t) / 1e6:13.1f} "
          f"{sum(d['dram__bytes_write.sum']) / len(t) / 1e6:14.1f}")
