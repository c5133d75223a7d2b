import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from mch_inputs import random_medium
from oracle import Oracle
from paper_2503_01276_b200 import Homogenizer
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import g_err
d, n, M, L, N = 2, 32, 8, 3, 2
for seed in range(40 + d + N, 90 + d + N):
    kap, ids = random_medium(d, n, N, seed=seed)
    try:
        o = Oracle(d, n, M, L, 2, N, kap, ids, layout="block")
        for k in o.plan.all_vertices(): o.local_system(k)
        break
    except RuntimeError: continue
Go = o.effective_coeffs()
res = {}
for rtol in [1e-12, 1e-13, 1e-14]:
    with Homogenizer(d, n, N, M, L, 2, kap, ids, layout="block", rtol=rtol) as h:
        h.solve_all()
        res[rtol] = h.effective_coeffs()
        its = [h.level_iterations(l).max() for l in range(1, L + 1)]
    errs = [g_err(res[rtol][i], Go[i]) for i in range(len(Go))]
    print(rtol, "max err vs oracle", max(errs), "at", int(np.argmax(errs)), "iters", its)
print("gpu 1e-12 vs 1e-14", max(g_err(res[1e-12][i], res[1e-14][i]) for i in range(len(Go))))
print("berr oracle", max(o.solve(k)["berr"] for k in o.plan.all_vertices()))
with Homogenizer(d, n, N, M, L, 2, kap, ids, layout="block", keep_all=True) as h:
    h.solve_all()
    Gg = h.effective_coeffs()
    for k in o.plan.all_vertices():
        i = o.plan.linear_index(k)
        e = g_err(Gg[i], Go[i])
        r = o.solve(k)
        pe = max(np.linalg.norm(h.local_solution(k, a) - r["phi"][a]) / np.linalg.norm(r["phi"][a]) for a in range(o.n_rhs))
        if e > 1e-9 or pe > 1e-8:
            print(k, "level", o.plan.level_of(k), "G err %.2e phi err %.2e" % (e, pe), "parents", o.plan.parents(k))
