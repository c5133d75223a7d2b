"""Turn the outputs of tools/r02b_profiles.sh in gpurun_out/ into the tracked summaries under
profiles/ (dev tool): launch list, DRAM bytes per PCG / transport launch (bench.py's `traffic`),
ncu summaries with the top source lines, the bench line."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02b"

rows = list(csv.reader(open(os.path.join(G, "launches_c5.csv"))))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    L.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
out, tot, pcg, tr = [], 0.0, [], []
for (i, k), m in L.items():
    t = m["gpu__time_duration.sum"] / 1e6
    d = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot += t
    out.append(f"{i:>4} {k[:60]:60s} {t:9.3f} ms  dram {d / 1e9:8.3f} GB")
    if "pcg" in k and "setup" not in k:
        pcg.append(d)
    if "transport" in k:
        tr.append(d)
out.append(f"total {tot:.3f} ms (ncu serialised, cold caches per launch)")
open(os.path.join(P, f"{tag}_launches_c5.txt"), "w").write(
    "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
    "python tools/run_config.py 5 1 (one B200)\n" + "\n".join(out) + "\n")
dj = {f"dram_bytes_pcg_L{i + 1}_launch": b for i, b in enumerate(pcg[:4])}
dj.update({f"dram_bytes_transport_L{i + 2}_launch": b for i, b in enumerate(tr[:3])})
json.dump({"c5": dj, "how": f"ncu dram__bytes_read.sum + dram__bytes_write.sum of each level's PCG and transport "
                            f"launch, profiles/{tag}_launches_c5.txt"},
          open(os.path.join(P, "r02_dram_per_launch.json"), "w"), indent=1)
for f in sorted(os.listdir(G)):
    if f.endswith("_summary.txt") and os.path.exists(os.path.join(G, f[:-12] + "_src.csv.gz")):
        name = f[:-12]
        if name not in ("fine3d_l4", "w7_l4", "pcg3d13_l3", "pcg3dc25_l2", "l1c_l1", "combine_l3"):
            continue
        summ = open(os.path.join(G, f)).read()
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                                os.path.join(G, name + "_src.csv.gz"), "18"], capture_output=True, text=True).stdout
        open(os.path.join(P, f"{tag}_{name}_ncu_c5.txt"), "w").write(
            "# ncu --set full --clock-control none --import-source on, one launch, config 5 (one B200)\n" + summ +
            "top source lines (share of warp instructions, share of stall samples) and SASS mix:\n" + lines)
b = os.path.join(G, "bench.json")
if os.path.exists(b):
    open(os.path.join(P, f"{tag}_bench_c5.json"), "w").write(open(b).read().strip().splitlines()[-1] + "\n")
print(sorted(f for f in os.listdir(P) if f.startswith(tag)))
