"""Summarise gpurun_out/launches_bench.csv (ncu --metrics gpu__time_duration.sum --clock-control none
-c 900 --csv of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-others`) into
profiles/r02c_launches_bench.txt: device time summed per kernel and its share (dev tool)."""
import collections
import csv
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", "launches_bench.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
L = [(r[ki], float(r[vi].replace(",", "")) / 1e6) for r in rows[hi + 1:] if len(r) > vi]
agg = collections.OrderedDict()
for k, t in L:
    a = agg.setdefault(re.sub(r"\(.*", "", k).replace("void ", ""), [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(a[1] for a in agg.values())
out = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 900, python bench.py --steps 2 --warmup 3 "
       "--no-cpu-baseline --no-others (one B200)",
       "# every launch of the run (3 warm-up + 2 timed steps, the e2e leg's steps, L2 flushes, peak probes), summed per "
       "kernel; share of the summed device time",
       f"# launches {len(L)}, summed {tot:.1f} ms (serialised, cold caches)"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k[:70]:70s} launches {n:4d}  {t:10.3f} ms  {100 * t / tot:5.1f}%")
open(os.path.join(ROOT, "profiles", "r02c_launches_bench.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:10]))
