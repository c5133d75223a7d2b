"""Per-problem PCG iteration counts of one level of a BASELINE config (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cid, lev = int(sys.argv[1]), int(sys.argv[2])
cfg = CONFIGS[cid]
kap, ids = make_medium(cfg)
with Homogenizer.from_config(cfg, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
    for l in range(1, lev + 1):
        h.solve_level(l)
    it = h.level_iterations(lev)
    pts = h.level_macropoints(lev)
    mx = it.max(axis=1)
    order = np.argsort(-mx)
    print("level", lev, "problems", it.size, "mean", it.mean(), "max", it.max())
    print("hist of per-macropoint max:", np.histogram(mx, bins=[0, 50, 100, 150, 200, 300, 1000])[0].tolist())
    mv = cfg.M + 1
    for i in order[:12]:
        m = int(pts[i]); k = (m % mv, (m // mv) % mv, m // (mv * mv))
        print(k, it[i].tolist())
