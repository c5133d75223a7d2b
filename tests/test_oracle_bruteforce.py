"""P1: oracle (sparse KKT + LU) vs dense brute force (quadrature + null-space method) on tiny
grids, levels 1 and 2 (BASELINE north_star "dense brute-force solves on
8×8 grids must agree")."""
import numpy as np
import pytest

from mch_inputs import periodic_medium, random_medium
from oracle import Oracle
from tests.bruteforce import BruteForce


def _find_medium(d, n, M, N, seed0):
    # every continuum must be present in every K_p (reading R13); scan seeds deterministically
    for seed in range(seed0, seed0 + 50):
        kap, ids = random_medium(d, n, N, seed=seed)
        try:
            o = Oracle(d, n, M, 1, 2, N, kap, ids)
            for k in o.plan.all_vertices():
                o.local_system(k)
            return kap, ids
        except RuntimeError:
            continue
    raise AssertionError("no admissible medium")


@pytest.mark.parametrize("d,n,M,L,N", [(2, 16, 4, 1, 2), (2, 16, 4, 2, 2), (2, 32, 4, 2, 3),
                                       (3, 16, 4, 2, 2)])
def test_oracle_equals_dense_bruteforce(d, n, M, L, N):
    kap, ids = _find_medium(d, n, M, N, seed0=10 * d + N)
    o = Oracle(d, n, M, L, 2, N, kap, ids)
    bf = BruteForce(d, n, M, L, 2, N, kap, ids)
    pts = list(o.plan.all_vertices())
    if d == 3:  # corner, edge, face, interior points of both levels (parents solved on demand)
        pts = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (2, 2, 2), (1, 1, 1), (3, 2, 1), (4, 4, 4)]
    for k in pts:
        ro = o.solve(k)
        rb = bf.solve(k)
        Go, Gb = ro["G"], rb["G"]
        scale = np.sqrt(np.outer(np.diag(Gb), np.diag(Gb))) + 1e-300
        assert np.max(np.abs(Go - Gb) / np.maximum(np.abs(Gb), scale)) < 1e-10, k
        po = ro["phi"].reshape(o.n_rhs, -1).T
        assert np.abs(po - rb["phi"]).max() / np.abs(rb["phi"]).max() < 1e-10, k


def test_rank_deficient_level_constraints():
    """Reading R20: a level mesh equal to the period of a centred inclusion (level 3, mesh 4h,
    period 4h) makes the two continuum rows of a subcell proportional in V_3; oracle (eigen
    truncation + KKT) equals the brute force (least squares + null space)."""
    kap, ids = periodic_medium(2, 64, 4, 0.3, 1.0, 30.0)
    o = Oracle(2, 64, 8, 3, 2, 2, kap, ids)
    bf = BruteForce(2, 64, 8, 3, 2, 2, kap, ids)
    for k in [(1, 0), (1, 1), (3, 2), (0, 1), (2, 1), (7, 8), (5, 3)]:
        ro, rb = o.solve(k), bf.solve(k)
        assert ro["level"] == 3
        Go, Gb = ro["G"], rb["G"]
        scale = np.sqrt(np.outer(np.diag(Gb), np.diag(Gb))) + 1e-300
        assert np.max(np.abs(Go - Gb) / np.maximum(np.abs(Gb), scale)) < 1e-9, k
        po = ro["phi"].reshape(o.n_rhs, -1).T
        assert np.abs(po - rb["phi"]).max() / np.abs(rb["phi"]).max() < 1e-9, k


@pytest.mark.parametrize("d,n,M,L,N", [(2, 16, 4, 1, 2), (2, 24, 6, 2, 2), (2, 64, 8, 3, 2),
                                       (3, 12, 3, 1, 2)])
def test_block_layout_oracle_equals_dense_bruteforce(d, n, M, L, N):
    """P1 for the block-centred layout (NEXT-1): x_p at block centres, K_p the
    block, subcells the blocks of R_p^+, T_n of Figure 2 — oracle vs the independent dense solver,
    every macropoint (3D: a sample)."""
    for seed in range(40 + d + N, 90 + d + N):
        kap, ids = random_medium(d, n, N, seed=seed)
        try:
            o = Oracle(d, n, M, L, 2, N, kap, ids, layout="block")
            for k in o.plan.all_vertices():
                o.local_system(k)
            break
        except RuntimeError:
            continue
    bf = BruteForce(d, n, M, L, 2, N, kap, ids, layout="block")
    pts = list(o.plan.all_vertices())
    if d == 3:
        pts = [(0, 0, 0), (1, 0, 0), (1, 1, 1), (2, 1, 0)]
    for k in pts:
        ro, rb = o.solve(k), bf.solve(k)
        Go, Gb = ro["G"], rb["G"]
        scale = np.sqrt(np.outer(np.diag(Gb), np.diag(Gb))) + 1e-300
        assert np.max(np.abs(Go - Gb) / np.maximum(np.abs(Gb), scale)) < 1e-10, k
        po = ro["phi"].reshape(o.n_rhs, -1).T
        assert np.abs(po - rb["phi"]).max() / np.abs(rb["phi"]).max() < 1e-10, k


@pytest.mark.parametrize("d,n,M,L,N", [(2, 32, 8, 2, 2), (2, 32, 8, 2, 1), (2, 64, 8, 3, 2)])
def test_physical_transport_oracle_equals_dense_bruteforce(d, n, M, L, N):
    """NEXT-4: nearest-S_1 parent evaluated at PHYSICAL
    coordinates, level-1 windows enlarged by η^{L-1}/2 layers so they contain every assigned
    child's window — oracle vs the independent dense solver at every macropoint (L = 3: a sample
    of each level)."""
    kap, ids = _find_medium(d, n, M, N, seed0=70 + d + N)
    o = Oracle(d, n, M, L, 2, N, kap, ids, interp="physical_s1")
    bf = BruteForce(d, n, M, L, 2, N, kap, ids, physical=True)
    pts = list(o.plan.all_vertices())
    if L == 3:
        pts = [(0, 0), (4, 4), (8, 0), (2, 0), (2, 2), (6, 4), (1, 0), (3, 1), (7, 7), (5, 6)]
    for k in pts:
        ro, rb = o.solve(k), bf.solve(k)
        Go, Gb = ro["G"], rb["G"]
        dg = np.abs(np.diag(Gb))
        scale = np.sqrt(np.outer(dg, dg)) + 1e-300
        null = dg <= 1e-9 * dg.max()  # N = 1: the phi_0 row is zero (P3)
        err = np.abs(Go - Gb) / np.maximum(np.abs(Gb), scale)
        err[null, :] = 0.0
        err[:, null] = 0.0
        assert np.max(err) < 1e-10, k
        assert np.max(np.abs(Go[null])) <= 1e-9 * dg.max() if null.any() else True
        po = ro["phi"].reshape(o.n_rhs, -1).T
        assert np.abs(po - rb["phi"]).max() / np.abs(rb["phi"]).max() < 1e-10, k


def test_physical_transport_windows_and_invariants():
    """NEXT-4 planner: level-1 windows carry l + η^{L-1}/2 layers and contain the windows of their
    children; the parent is the nearest S_1 point; partition of unity (P3) and the constraint
    targets of the combined φ (P7) hold at every child."""
    d, n, M, L, N = 2, 64, 8, 3, 2
    kap, ids = _find_medium(d, n, M, N, seed0=90)
    o = Oracle(d, n, M, L, 2, N, kap, ids, interp="physical_s1")
    pl = o.plan
    for k in pl.all_vertices():
        lo, hi = pl.window(k)
        if pl.level_of(k) == 1:
            assert pl.l_of(k) == 3
            continue
        (t, w), = pl.parents(k)
        assert w == 1.0 and pl.level_of(t) == 1
        assert max(abs(t[i] - k[i]) for i in range(d)) <= 2
        plo, phi = pl.window(t)
        assert all(plo[i] <= lo[i] and phi[i] >= hi[i] for i in range(d))
    for k in [(2, 0), (6, 4), (3, 1), (5, 6)]:
        r = o.solve(k)
        S = o.local_system(k)
        phi = r["phi"].reshape(o.n_rhs, -1)
        assert np.abs(phi[:N].sum(axis=0) - 1.0).max() < 1e-10           # P3
        cons = S["C1"] @ phi.T                                               # P7: original targets
        act = S["active"]
        assert np.abs(cons[act] - S["g0"][act]).max() <= 1e-10 * np.abs(S["g0"]).max()
