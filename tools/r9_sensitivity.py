"""NEXT-4: how sensitive the effective coefficients are to reading R9 (dev/measurement tool).
Runs a BASELINE 2D config with nearest-S_1 parents in local coordinates (R9, MCH_INTERP_NEAREST_S1)
and in physical coordinates with enlarged level-1 windows (MCH_INTERP_PHYSICAL_S1), and the plain
method (L = 1, every macropoint on the fine mesh); prints per level the relative difference of G
(Frobenius per macropoint, median / max) between the readings and against the plain method."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from mch_inputs import CONFIGS, make_medium  # noqa: E402
from paper_2503_01276_b200 import Homogenizer  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = CONFIGS[cid]
kap, ids = make_medium(cfg)
kd, idd = torch.from_numpy(kap).cuda(), torch.from_numpy(ids).cuda()
out, lev_of = {}, None
for name, interp, L in (("R9_local", "nearest_s1", cfg.L), ("physical", "physical_s1", cfg.L),
                        ("R9_R10_dlinear", "dlinear", cfg.L), ("plain", "dlinear", 1)):
    t0 = time.time()
    with Homogenizer(cfg.d, cfg.n, cfg.N, cfg.M, L, cfg.eta, kd, idd, interp=interp) as h:
        h.solve_all()
        torch.cuda.synchronize()
        out[name] = h.effective_coeffs()
        ms = [h.level_stats(l)["ms_total"] for l in range(1, L + 1)]
        if L == cfg.L and lev_of is None:
            lev_of = np.zeros(h.num_macropoints, dtype=int)
            for l in range(1, L + 1):
                lev_of[h.level_macropoints(l)] = l
    print(f"{name}: levels ms {[round(m, 2) for m in ms]} wall {time.time() - t0:.1f}s", flush=True)


def rel(a, b):
    return np.linalg.norm((a - b).reshape(len(a), -1), axis=1) / np.linalg.norm(b.reshape(len(b), -1), axis=1)


res = {"config": cfg.name}
for lev in range(1, cfg.L + 1):
    m = lev_of == lev
    d_rp = rel(out["physical"][m], out["R9_local"][m])
    d_lp = rel(out["R9_local"][m], out["plain"][m])
    d_pp = rel(out["physical"][m], out["plain"][m])
    d_dp = rel(out["R9_R10_dlinear"][m], out["plain"][m])
    res[f"level{lev}"] = {"macropoints": int(m.sum()),
                          "physical_vs_R9_median": float(np.median(d_rp)), "physical_vs_R9_max": float(d_rp.max()),
                          "R9_vs_plain_median": float(np.median(d_lp)), "physical_vs_plain_median": float(np.median(d_pp)),
                          "dlinear_R9_vs_plain_median": float(np.median(d_dp))}
print(json.dumps(res))
