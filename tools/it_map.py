"""Mean PCG iterations per level-1 window of a config, laid out on the T_1 lattice (dev tool)."""
import sys; sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200 import Homogenizer
cfg = CONFIGS[int(sys.argv[1])]
kap, ids = make_medium(cfg)
with Homogenizer.from_config(cfg, kap, ids) as h:
    h.solve_level(1)
    it = h.level_iterations(1)
    pts = h.level_macropoints(1)
    ks = [(p % h.mv, p // h.mv) for p in pts]
    xs = sorted(set(k[0] for k in ks))
    grid = np.zeros((len(xs), len(xs)))
    for (kx, ky), v in zip(ks, it.mean(axis=1)):
        grid[xs.index(ky), xs.index(kx)] = v
    np.set_printoptions(linewidth=200)
    print(grid.round(0).astype(int))
