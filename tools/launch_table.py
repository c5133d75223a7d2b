"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    L.setdefault((r[ii], r[ki][:48]), {})[r[mi]] = float(r[vi].replace(",", ""))
tot = 0.0
for (i, k), m in L.items():
    t = m["gpu__time_duration.sum"] / 1e6
    tot += t
    d = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{i:>4} {k:48s} {t:9.3f} ms  dram {d:8.2f} GB")
print(f"total {tot:.3f} ms")
