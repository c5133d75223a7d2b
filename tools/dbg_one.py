import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mch_inputs import random_medium
from paper_2503_01276_b200 import Homogenizer
d, n, M, L, N, seed = 2, 32, 4, 1, 2, 13
kap, ids = random_medium(d, n, N, seed=seed)
try:
    with Homogenizer(d, n, N, M, L, 2, kap, ids, max_iter=300) as h:
        h.solve_level(1)
except Exception as e:
    print("ERR", str(e)[:200])
