import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from mch_inputs import random_medium
from paper_2503_01276_b200 import Homogenizer
from paper_2503_01276_b200._native import MchError
for (d, n, M, L, N, seed) in [(2, 32, 4, 2, 3, 13), (2, 32, 4, 1, 3, 13), (2, 32, 4, 1, 2, 13), (2, 64, 8, 1, 2, 7), (2, 64, 8, 1, 3, 7)]:
    kap, ids = random_medium(d, n, N, seed=seed)
    for mode in ["", "gn", "old"]:
        if mode: os.environ["MCH_PCG"] = mode
        else: os.environ.pop("MCH_PCG", None)
        try:
            with Homogenizer(d, n, N, M, L, 2, kap, ids, max_iter=3000) as h:
                h.solve_level(1)
                it = h.level_iterations(1)
                print(d, n, M, L, N, seed, mode or "l1op", "iters max", it.max(), "mean", round(it.mean(), 1), flush=True)
        except MchError as e:
            print(d, n, M, L, N, seed, mode or "l1op", "ERR", str(e)[:160], flush=True)
