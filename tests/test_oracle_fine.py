"""Pins for oracle/fine.py (NEXT-3: fine reference solve, block averages, e₂)."""
import numpy as np
import pytest

from mch_inputs import random_medium
from oracle.fine import (cell_means, e2, fine_block_averages, fine_load, fine_solve,
                         macro_block_averages)


def _centres(n, d):
    c = (np.arange(n) + 0.5) / n
    return np.meshgrid(*([c] * d), indexing="ij")[::-1]  # x_0 .. x_{d-1}, arrays [.., y, x]


@pytest.mark.parametrize("d,ns", [(2, [16, 32, 64]), (3, [8, 16])])
def test_fine_solve_manufactured_rate(d, ns):
    """κ ≡ 2.5, u = Π sin(πx_i): f = 2.5 dπ² u at cell centres; nodal max error O(h²)."""
    errs = []
    for n in ns:
        xs = _centres(n, d)
        f = 2.5 * d * np.pi ** 2 * np.prod([np.sin(np.pi * x) for x in xs], axis=0)
        u = fine_solve(np.full((n,) * d, 2.5), f)
        g = np.linspace(0, 1, n + 1)
        nodes = np.meshgrid(*([g] * d), indexing="ij")[::-1]
        ex = np.prod([np.sin(np.pi * x) for x in nodes], axis=0)
        errs.append(np.abs(u - ex).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates.min() > 1.8, (errs, rates)


def test_fine_solve_maximum_principle_and_boundary():
    """Q1 on squares is an M-matrix: f ≥ 0 ⇒ u ≥ 0; u = 0 on ∂Ω; f ≡ 0 ⇒ u ≡ 0."""
    kap, ids = random_medium(2, 24, 2, seed=4)
    u = fine_solve(kap, np.ones((24, 24)))
    assert u.min() >= 0.0 and u[0].max() == 0 and u[-1].max() == 0 and u[:, 0].max() == 0
    assert np.abs(fine_solve(kap, np.zeros((24, 24)))).max() == 0.0


def test_fine_load_total():
    """Σ_a F_a = ∫ f (partition of unity)."""
    f = np.random.default_rng(0).uniform(size=(8, 8, 8))
    assert abs(fine_load(f).sum() - f.sum() / 8 ** 3) < 1e-14


def test_block_averages_linear_field():
    """u = x_0 (Q1 exact): cell means = centre values, so ū_{p,i} = mean x_0 over the cells of
    continuum i in K_p, computed here by brute force over cell centres."""
    d, n, M, N = 2, 16, 4, 2
    _, ids = random_medium(d, n, N, seed=2)
    g = np.linspace(0, 1, n + 1)
    u = np.broadcast_to(g[None, :], (n + 1, n + 1)).copy()
    ub = fine_block_averages(u, ids, N, M)
    xc = (np.arange(n) + 0.5) / n
    c = n // M
    for p in range(M * M):
        kx, ky = p % M, p // M
        for i in range(N):
            vals = [xc[x] for y in range(ky * c, ky * c + c) for x in range(kx * c, kx * c + c) if ids[y, x] == i]
            assert abs(ub[p, i] - np.mean(vals)) < 1e-14
    assert np.allclose(cell_means(u)[0], xc)


def test_macro_block_average_and_e2():
    """bilinear U: block mean = value at the block centre; e₂ of ū(1+δ) against ū is |δ|."""
    M = 4
    g = np.linspace(0, 1, M + 1)
    X, Y = np.meshgrid(g, g)
    U = np.stack([(X + 2 * Y).reshape(-1), (X * Y).reshape(-1)])
    Ub = macro_block_averages(U, 2, M)
    for p in range(M * M):
        cx, cy = (p % M + 0.5) / M, (p // M + 0.5) / M
        assert abs(Ub[p, 0] - (cx + 2 * cy)) < 1e-14 and abs(Ub[p, 1] - cx * cy) < 1e-14
    ub = np.random.default_rng(1).uniform(1, 2, size=(16, 2))
    assert np.allclose(e2(ub * 1.03, ub), 0.03, rtol=1e-12)


def test_host_validate_matches_oracle():
    """the product's host post-processing (validate.py) against the oracle's formulas"""
    from paper_2503_01276_b200.validate import macro_block_averages as mba, relative_l2_error
    rng = np.random.default_rng(0)
    for d, M, N in ((2, 8, 3), (3, 4, 2)):
        U = rng.normal(size=(N, (M + 1) ** d))
        assert np.abs(mba(U, d, M) - macro_block_averages(U, d, M)).max() < 1e-15
    ub = rng.uniform(1, 2, size=(20, 2))
    ub[3, 1] = np.nan
    Ub = ub + rng.normal(size=ub.shape) * 0.01
    assert np.allclose(relative_l2_error(Ub, ub), e2(Ub, ub), rtol=1e-14)
