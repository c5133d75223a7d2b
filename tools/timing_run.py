import sys, os; sys.path.insert(0,'/root/repo')
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cfg=CONFIGS[2]
kap,ids=make_medium(cfg)
with Homogenizer(2, cfg.n, cfg.N, cfg.M, 1, 2, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
    h.solve_level(1)
