"""Per-RHS and per-window-size PCG iteration statistics of one config (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cfg = CONFIGS[int(sys.argv[1])]
kap, ids = make_medium(cfg)
with Homogenizer.from_config(cfg, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
    h.solve_all()
    for lev in range(1, cfg.L + 1):
        it = h.level_iterations(lev)
        pts = h.level_macropoints(lev)
        n = cfg.n // cfg.M
        sizes = []
        for m in pts:
            k = [(m // (cfg.M + 1) ** i) % (cfg.M + 1) for i in range(cfg.d)]
            ext = [min(cfg.n, (ki * n + 1.5 * n)) - max(0, ki * n - 1.5 * n) for ki in k]
            sizes.append(int(np.prod(ext)))
        sizes = np.array(sizes)
        print(f"L{lev}: problems {it.size} mean {it.mean():.1f} max {it.max()} per-rhs mean {np.round(it.mean(0),1)} max {it.max(0)}")
        for s in sorted(set(sizes)):
            sel = sizes == s
            print(f"   window cells {s}: {sel.sum()} mps, iters mean {it[sel].mean():.1f} max {it[sel].max()}")
        print("   per-macropoint max/mean ratio", np.round((it.max(1) / it.mean(1)).mean(), 2))
