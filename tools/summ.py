"""Summarise run_config logs (last rep) and the pytest tail."""
import json, sys
for f in sys.argv[1:]:
    print("==", f)
    lines = open(f).read().splitlines()
    reps = sorted({l.split()[0] for l in lines if l.startswith("rep")})
    for l in lines:
        if not l.startswith(reps[-1] if reps else "rep"):
            continue
        if "wall" in l:
            print(l)
            continue
        lv, js = l.split(": ", 1)
        d = json.loads(js)
        print(lv, "ms", d["ms_total"], "pcg", d["ms_pcg"], "setup", d["ms_setup"], "gram", d["ms_gram"],
              "iters", round(d["avg_iters"], 1), "max", d["iters_max"])
