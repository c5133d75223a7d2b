"""Solve one BASELINE config once (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
kap, ids = make_medium(cfg)
with Homogenizer.from_config(cfg, torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()) as h:
    h.solve_all()
    print([round(h.level_stats(l)["ms_pcg"], 2) for l in range(1, cfg.L + 1)])
