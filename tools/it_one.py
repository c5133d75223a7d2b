import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cfg=CONFIGS[2]
kap,ids=make_medium(cfg)
for mode in (None, "old"):
    import os
    if mode: os.environ["MCH_PCG"]=mode
    with Homogenizer(2, cfg.n, cfg.N, cfg.M, 1, 2, kap, ids) as h:
        h.solve_level(1)
        it=h.level_iterations(1)
        pts=h.level_macropoints(1)
        i=pts.index(h.linear_index((16,16)))
        print(mode, "window (16,16) iterations per rhs:", it[i].tolist(), "mean all", it.mean().round(1))
