"""Per-source-line instruction and stall shares of an ncu report (first kernel), plus SASS opcode mix."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if rep.endswith(".csv.gz"):  # an exported source page (ncu -i ... --page source --csv | gzip)
    import gzip
    src = gzip.open(rep, "rt").read()
else:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
cur = None
per_i, per_s, text, ops = collections.Counter(), collections.Counter(), {}, collections.Counter()
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:
        key = (cur, int(r[0]))
        text[key] = r[1].strip()[:90]
        try:
            per_i[key] += int(r[7]); per_s[key] += int(r[4])
        except (ValueError, IndexError):
            pass
    else:
        t = r[3].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        try:
            ops[op.split(".")[0]] += int(r[7])
        except (ValueError, IndexError):
            pass
ti, ts = sum(per_i.values()) or 1, sum(per_s.values()) or 1
print("warp instructions", ti, "stall samples", ts)
for k, v in per_i.most_common(top):
    print(f"{100*v/ti:5.1f}% inst {100*per_s[k]/ts:5.1f}% stall  {k[0]}:{k[1]}  {text.get(k, '')}")
print(" ".join(f"{k}:{100*v/ti:.1f}%" for k, v in ops.most_common(25)))
