"""Summarise an ncu report: key raw metrics per launch and top source lines by stall samples."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]
idx = {k: h.index(k) for k in keys if k in h}
for r in rows[2:]:
    print(" | ".join(f"{k.split('.')[0].replace('smsp__pcsamp_warps_issue_stalled_','stall_')}={r[i]}{units[i] if units[i] not in ('','inst') else ''}" for k, i in idx.items()))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
per = collections.Counter(); text = {}; cur = None; last = None
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    try: ln = int(r[0]) if r[0] else None
    except ValueError: ln = None
    if ln is not None: last = (cur, ln); text[last] = r[1].strip()[:100]
    try: per[last] += int(r[4])
    except (ValueError, IndexError): pass
tot = sum(per.values()) or 1
print("stall samples", tot)
for k, v in per.most_common(top): print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]}  {text.get(k,'')}")
