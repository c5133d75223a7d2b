import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mch_inputs import random_medium
from paper_2503_01276_b200 import Homogenizer
d, n, M, L, N = 2, 16, 4, 1, 2
kap, ids = random_medium(d, n, N, seed=22)
try:
    with Homogenizer(d, n, N, M, L, 2, kap, ids) as h:
        h.solve_all()
        print("ok", h.level_iterations(1).max())
except Exception as e:
    print("ERR", str(e)[:300])
