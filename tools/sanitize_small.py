"""Tiny 2D/3D runs covering every kernel variant of the hot path, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_small.py [variant ...]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from mch_inputs import random_medium  # noqa: E402
from paper_2503_01276_b200 import Homogenizer  # noqa: E402

CASES = {
    "2d": (2, 64, 2, 8, 3, 11),      # k_pcg2d level-1 / 49 / 25 variants, 2D transport, coarse space
    "3d_small": (3, 16, 2, 4, 2, 12),  # k_pcg3d_l1c (cluster), fused fine passes, k_pcg3d_w7
    "3d_13": (3, 32, 2, 4, 2, 13),   # k_pcg3d <13>, fused fine passes with 8 cells per H
}
for name in (sys.argv[1:] or list(CASES)):
    d, n, N, M, L, seed = CASES[name]
    for s in range(seed, seed + 40):
        kap, ids = random_medium(d, n, N, seed=s)
        try:
            with Homogenizer(d, n, N, M, L, 2, kap, ids) as h:
                h.solve_all()
                G = h.effective_coeffs()
            break
        except RuntimeError as e:
            if "ERANK" not in str(e):
                raise
    print(name, "ok", np.isfinite(G).all(), flush=True)
