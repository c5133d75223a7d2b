"""Write the oracle's results for full-size 3D interior windows (TEST INFRASTRUCTURE).

Calls only ``oracle/`` and ``mch_inputs`` (no CUDA path).  The oracle's sparse LU of an
unclipped 49³-node level-1 window costs ≈ 100 s and ≈ 3 GB, too slow to
repeat inside every GPU test run, so the GPU parity test (`tests/test_gpu_parity.py::
test_config_interior_3d`) reads these stored values.  For each sampled macropoint the file holds
the Eq. (7) Gram matrix G and the fine combined local solution φ_p
(Eq. 11) on the window nodes whose local indices are all even (a 25³ sub-lattice
of the 49³ window: the ℓ₂ parity bar is evaluated on that sample), plus a digest of the medium so
a changed generator invalidates the cache.

Samples (VERDICT r01 "next round" 1): config 4 — the interior level-1 point (4,4,4) and the
interior level-2 children (3,3,3) (eight interior parents) and (3,4,4) (two); config 5 — the
interior chain (8,8,8) [L1] → (4,4,4) [L2] → (6,6,6) [L3] → (7,7,7) [L4] (27 subcells, 54
constraint rows, unclipped 49³ fine windows at every level).

    python tests/golden/make_oracle_cache.py [c4|c5 ...]
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from mch_inputs import CONFIGS, make_medium  # noqa: E402
from oracle import Oracle  # noqa: E402
from oracle.hmh import run_parallel  # noqa: E402

SAMPLES = {
    4: [(4, 4, 4), (3, 3, 3), (3, 4, 4)],
    5: [(8, 8, 8), (4, 4, 4), (6, 6, 6), (7, 7, 7)],
}
STRIDE = 2


def medium_digest(kap, ids) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(kap).tobytes())
    h.update(np.ascontiguousarray(ids).tobytes())
    return h.hexdigest()[:32]


def ancestors(o, k, acc):
    k = tuple(k)
    if k in acc:
        return
    acc.add(k)
    for t, _ in o.plan.parents(k):
        ancestors(o, t, acc)


def main(cids):
    for cid in cids:
        cfg = CONFIGS[cid]
        kap, ids = make_medium(cfg)
        o = Oracle.from_config(cfg, kap, ids)
        need = set()
        for k in SAMPLES[cid]:
            ancestors(o, k, need)
        by_level = [[k for k in sorted(need) if o.plan.level_of(k) == lev] for lev in range(1, cfg.L + 1)]
        t0 = time.time()
        walls, used = run_parallel(o, by_level, workers=min(8, len(os.sched_getaffinity(0))), keep_phi=True)
        out = {"digest": np.array(medium_digest(kap, ids)), "stride": np.array(STRIDE),
               "points": np.array(SAMPLES[cid], dtype=np.int64)}
        for k in SAMPLES[cid]:
            r = o.solve(k)
            tag = "_".join(str(v) for v in k)
            out[f"G_{tag}"] = r["G"]
            out[f"phi_{tag}"] = np.ascontiguousarray(r["phi"][:, ::STRIDE, ::STRIDE, ::STRIDE])
            out[f"shape_{tag}"] = np.array(r["phi"].shape[1:], dtype=np.int64)
        path = os.path.join(HERE, f"oracle_cache_c{cid}.npz")
        np.savez_compressed(path, **out)
        print(f"c{cid}: {len(need)} oracle solves ({[len(b) for b in by_level]} per level), "
              f"{time.time() - t0:.0f} s on {used} workers -> {path}", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["c4", "c5"]
    main([int(a.lstrip("c")) for a in args])
