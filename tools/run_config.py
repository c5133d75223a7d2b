"""Run one BASELINE config through the C ABI and print per-level stats (dev tool)."""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch

from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer

cid = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[cid]
t0 = time.time()
kap, ids = make_medium(cfg)
print(f"config {cid}: medium {time.time()-t0:.1f}s", flush=True)
kd = torch.from_numpy(kap).cuda()
idd = torch.from_numpy(ids).cuda()
for rep in range(reps):
    torch.cuda.synchronize()
    t0 = time.time()
    with Homogenizer.from_config(cfg, kd, idd) as h:
        h.solve_all()
        G = h.effective_coeffs()
        torch.cuda.synchronize()
        wall = time.time() - t0
        for l in range(1, cfg.L + 1):
            s = h.level_stats(l)
            s["mp_per_s"] = s["macropoints"] / (s["ms_total"] * 1e-3)
            s["pcg_GBps"] = s["pcg_bytes"] / (s["ms_pcg"] * 1e-3) / 1e9
            s["avg_iters"] = s["iters_total"] / max(1, s["problems"])
            print(f"rep{rep} L{l}: " + json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in s.items()}), flush=True)
    print(f"rep{rep} wall {wall:.3f}s  G finite {np.isfinite(G).all()}  |G|max {np.abs(G).max():.4e}", flush=True)
