"""A/B of one developer switch (dev tool): runs a BASELINE config twice in child processes, without
and with VAR=VALUE, and prints the per-level device time and the max relative difference of G.
usage: env_ab.py <config> VAR=VALUE"""
import os
import subprocess
import sys

if len(sys.argv) > 3 and sys.argv[2] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    from mch_inputs import CONFIGS, make_medium
    from paper_2503_01276_b200 import Homogenizer
    cfg = CONFIGS[int(sys.argv[1])]
    kap, ids = make_medium(cfg)
    with Homogenizer.from_config(cfg, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
        for rep in range(2):
            h.reset()
            h.solve_all()
        print("  " + "  ".join(f"L{l} {h.level_stats(l)['ms_total']:.3f} ms" for l in range(1, cfg.L + 1)), flush=True)
        np.save(sys.argv[3], np.asarray(h.effective_coeffs()))
    sys.exit(0)

import numpy as np

cid, kv = sys.argv[1], sys.argv[2]
var, val = kv.split("=", 1)
outs = []
for i, extra in enumerate(({}, {var: val})):
    env = dict(os.environ, **extra)
    out = f"/tmp/env_ab_{i}.npy"
    print(f"config {cid} {'default' if not extra else kv}", flush=True)
    subprocess.run([sys.executable, __file__, cid, "child", out], env=env, check=True)
    outs.append(np.load(out))
a, b = outs
print("max rel dG", float(np.max(np.abs(a - b)) / np.max(np.abs(a))), "bitwise equal", bool(np.array_equal(a, b)))
