"""Type 1/2/3 errors on the paper's Example-1 medium, on the GPU (dev tool).

Layered κ = g1·g2 with ε = 1/48 (reading R25), source f of PAPER.md:516-528, h = 1/960, block
layout, R_p = K_p, η = 2.  Differences from the paper's runs: oversampling l = 1, 2 (the paper uses
⌈−2 ln H⌉; the local solvers here take l ≤ 2) and local-coordinate transport (reading R9).
Prints one JSON line per H.
"""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np

from mch_inputs import paper_medium, paper_source
from paper_2503_01276_b200 import Homogenizer
from paper_2503_01276_b200.validate import macro_block_averages, relative_l2_error

d, n, N, eps = 2, 960, 2, 1.0 / 48
kap, ids = paper_medium(d, n, eps)
f = paper_source(d, n, ids, eps)
t0 = time.time()
with Homogenizer(d, n, N, 12, 1, 2, kap, ids, layout="block") as h:
    u, fit = h.fine_solve(f, rtol=1e-10)
t_fine = time.time() - t0
print(json.dumps({"fine_solve": {"n": n, "iterations": fit, "seconds": round(t_fine, 3)}}), flush=True)
for M, L, l in [tuple(int(v) for v in s.split(",")) for s in (sys.argv[1:] or ["12,3,1", "24,3,1", "12,3,2", "24,3,2"])]:
    U = {}
    for LL in (1, L):
        t0 = time.time()
        with Homogenizer(d, n, N, M, LL, 2, kap, ids, l=l, layout="block", max_iter=200000) as h:
            h.set_source(f)
            h.solve_all()
            Um, it = h.macro_solve(rtol=1e-12)
            U[LL] = macro_block_averages(Um, d, M)
            if LL == 1:
                ref = h.fine_block_averages(u)
        print(f"# H=1/{M} L={LL} l={l} {time.time() - t0:.2f}s", file=sys.stderr, flush=True)
    e = [relative_l2_error(U[1], ref), relative_l2_error(U[L], ref), relative_l2_error(U[L], U[1])]
    print(json.dumps({"H": f"1/{M}", "L": L, "l": l, "type1": e[0].tolist(), "type2": e[1].tolist(),
                      "type3": e[2].tolist()}), flush=True)
