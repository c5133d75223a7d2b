"""Per-rhs PCG iteration statistics of a BASELINE config (dev tool)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer

cid = int(sys.argv[1])
cfg = CONFIGS[cid]
kap, ids = make_medium(cfg)
with Homogenizer.from_config(cfg, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
    h.solve_all()
    for lev in range(1, cfg.L + 1):
        it = h.level_iterations(lev)
        print(f"c{cid} L{lev}: mean per rhs {np.round(it.mean(axis=0), 1).tolist()}  max per rhs {it.max(axis=0).tolist()}")
