"""Per-phase cycle counters of the 2D on-chip PCG (dev tool): build with MCH_BUILD_TIMING=1 and run
with MCH_PCG_TIMING=1 (and MCH_LIB pointing at lib/libmch_timing.so); prints one line per level.
usage: timing_run.py [config] [L]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
L = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.L
kap, ids = make_medium(cfg)
with Homogenizer(cfg.d, cfg.n, cfg.N, cfg.M, L, cfg.eta, torch.from_numpy(kap).cuda(),
                 torch.from_numpy(ids).cuda()) as h:
    h.solve_all()
