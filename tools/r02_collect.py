"""Turn the round-2 GPU outputs in gpurun_out/ into the tracked summaries under profiles/ (dev tool)."""
import collections
import csv
import gzip
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"


def launches(cfg="c5"):
    path = os.path.join(G, f"launches_{cfg}.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        L.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    out, tot, pcg = [], 0.0, []
    for (i, k), m in L.items():
        t = m["gpu__time_duration.sum"] / 1e6
        d = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        tot += t
        out.append(f"{i:>4} {k[:60]:60s} {t:9.3f} ms  dram {d / 1e9:8.3f} GB")
        if "pcg" in k and "setup" not in k:
            pcg.append(d)
    out.append(f"total {tot:.3f} ms (ncu serialised, cold caches per launch)")
    open(os.path.join(P, f"{tag}_launches_{cfg}.txt"), "w").write(
        f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
        f"python tools/run_config.py {cfg[1:]} 1 (one B200)\n" + "\n".join(out) + "\n")
    return pcg


def ncu_summary(name):
    raw = os.path.join(G, f"r02_{name}_raw.csv")
    if not os.path.exists(raw):
        return
    rows = list(csv.reader(open(raw)))
    if len(rows) < 3:
        return
    h, u, v = rows[0], rows[1], rows[2]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    lines = [f"# ncu --set full --clock-control none --import-source on, one launch, config 5 (one B200)"]
    for w in want:
        if w in h:
            i = h.index(w)
            lines.append(f"{w:70s} {v[i]:>24s} {u[i]}")
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines.append("stall reasons (warps per issue-active cycle):")
    for val, n in sorted(st, reverse=True)[:10]:
        lines.append(f"  {n:30s} {val:.3f}")
    src = os.path.join(G, f"r02_{name}_src.csv.gz")
    if os.path.exists(src):
        per, text, hdr, cur = collections.Counter(), {}, None, None
        for r in csv.reader(io.StringIO(gzip.open(src, "rt").read())):
            if not r:
                continue
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr and r[0].isdigit() and cur:
                try:
                    ie, isx = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
                    per[(cur, int(r[0]))] += float(r[ie] or 0)
                    text[(cur, int(r[0]))] = (r[1].strip()[:90], float(r[isx] or 0))
                except (ValueError, IndexError):
                    pass
        tot = sum(per.values()) or 1.0
        stot = sum(t[1] for t in text.values()) or 1.0
        lines.append("top source lines (share of warp instructions, share of stall samples):")
        for k, vv in per.most_common(15):
            lines.append(f"  {100 * vv / tot:5.1f}% inst {100 * text[k][1] / stot:5.1f}% stall  {k[0]}:{k[1]}  {text[k][0]}")
    open(os.path.join(P, f"{tag}_{name}_ncu_c5.txt"), "w").write("\n".join(lines) + "\n")


pcg = launches("c5")
for name in ("l1c", "pcg3dc25", "pcg3d13", "w7", "fine3d_l4", "pinv_l4"):
    ncu_summary(name)
if len(pcg) >= 4:
    json.dump({"c5": {f"dram_bytes_pcg_L{i + 1}_launch": b for i, b in enumerate(pcg[:4])},
               "how": "ncu dram__bytes_read.sum + dram__bytes_write.sum of each level's PCG launch, "
                      "profiles/" + tag + "_launches_c5.txt"},
              open(os.path.join(P, f"{tag}_dram_per_launch.json"), "w"), indent=1)
b = os.path.join(G, "bench.json")
if os.path.exists(b):
    open(os.path.join(P, f"{tag}_bench_c5.json"), "w").write(open(b).read().strip().splitlines()[-1] + "\n")
print(sorted(f for f in os.listdir(P) if f.startswith(tag)))
