"""A/B of the two-level preconditioner on the generic PCG at level 1 (dev tool):
MCH_PCG=old forces the generic kernel; MCH_COARSE=1 adds the coarse space.  Prints level-1
iterations, time and the max relative difference of G between the two runs."""
import os
import subprocess
import sys

if len(sys.argv) > 3 and sys.argv[2] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    from mch_inputs import CONFIGS, make_medium
    from paper_2503_01276_b200 import Homogenizer
    cfg = CONFIGS[int(sys.argv[1])]
    kap, ids = make_medium(cfg)
    with Homogenizer(cfg.d, cfg.n, cfg.N, cfg.M, 1, cfg.eta, torch.from_numpy(kap).cuda(),
                     torch.from_numpy(ids).cuda()) as h:
        for rep in range(2):
            h.reset()
            h.solve_level(1)
        st = h.level_stats(1)
        G = h.effective_coeffs()
        np.save(sys.argv[3], G)
        print(f"  iters mean {st['iters_total'] / st['problems']:.1f} max {st['iters_max']} pcg {st['ms_pcg']:.2f} ms "
              f"setup {st['ms_setup']:.2f} ms", flush=True)
    sys.exit(0)

cid = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "old"  # "old": generic k_pcg; "chip": on-chip k_pcg2d
for coarse in ("0", "1"):
    env = dict(os.environ, MCH_COARSE=coarse)
    if mode == "old":
        env["MCH_PCG"] = "old"
    print(f"config {cid} {mode} PCG, coarse={coarse}", flush=True)
    subprocess.run([sys.executable, __file__, cid, "child", f"/tmp/G_{coarse}.npy"], env=env, check=True)
import numpy as np
G0, G1 = np.load("/tmp/G_0.npy"), np.load("/tmp/G_1.npy")
sc = np.sqrt(np.abs(np.einsum("pii->pi", G0)))
den = np.maximum(np.abs(G0), sc[:, :, None] * sc[:, None, :]) + 1e-300
print("max rel dG", float((np.abs(G1 - G0) / den).max()))
