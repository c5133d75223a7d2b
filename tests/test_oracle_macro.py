"""Pins for oracle/macro.py (NEXT-2: load vectors and the upscaled system, Eqs. 6-7)."""
import numpy as np
import pytest

from mch_inputs import random_medium
from oracle import Oracle
from oracle.macro import block_operator, load_vectors, macro_solve


def test_load_vectors_partition_of_unity():
    """Σ_j φ_j ≡ 1 (P3) ⇒ Σ_j b_j = ∫_{K_p} f; with f ≡ 1, Σ_j b_j = |K_p| exactly"""
    kap, ids = random_medium(2, 32, 2, seed=11)
    for layout, M in (("vertex", 4), ("block", 4)):
        o = Oracle(2, 32, M, 2, 2, 2, kap, ids, layout=layout)
        b = load_vectors(o, np.ones((32, 32)))
        kp = []
        for k in o.plan.all_vertices():
            ext = 1.0
            for ki in k:
                lo = ki * o.plan.c - (o.plan.c // 2 if layout == "vertex" else 0)
                ext *= (min(32, lo + o.plan.c) - max(0, lo)) / 32.0
            kp.append(ext)
        assert np.abs(b.sum(axis=1) - np.array(kp)).max() < 1e-13


@pytest.mark.parametrize("d", [2, 3])
def test_macro_laplacian_manufactured_rate(d, omega=None):
    """G_p with only B^{mn} = δ_mn |K_p| and N = 1: the macro system is the Q1 Laplacian with
    block-midpoint quadrature.  Manufactured u = Π sin(ω_i π x_i), f = Σω_i² π² u, b = ∫_{K_p} f:
    the nodal max error decays at O(H²) (SPEC assemble_macro example).  ω = (1, 2[, 1]): with all
    ω_i equal the 2D rotated-stencil scheme is nodally exact for the mode (a closed form checked
    separately below), which would hide the rate."""
    errs = []
    om = omega or ([1, 2] if d == 2 else [1, 2, 1])
    Ms = [8, 16, 32] if d == 2 else [4, 8, 16]
    for M in Ms:
        H = 1.0 / M
        P = M ** d
        G = np.zeros((P, 1 + d, 1 + d))
        G[:, 1:, 1:] = np.eye(d) * H ** d
        # b = ∫_{K_p} f exactly (product of 1D integrals of sin)
        b = np.zeros((P, 1))
        for p in range(P):
            kb = [(p // M ** i) % M for i in range(d)]
            v = sum(w * w for w in om) * np.pi ** 2
            for i in range(d):
                w = om[i] * np.pi
                v *= (np.cos(w * kb[i] * H) - np.cos(w * (kb[i] + 1) * H)) / w
            b[p, 0] = v
        U = macro_solve(d, 1, M, G, b)[0]
        nv = M + 1
        ex = np.ones(nv ** d)
        for node in range(nv ** d):
            for i in range(d):
                ex[node] *= np.sin(om[i] * np.pi * ((node // nv ** i) % nv) * H)
        errs.append(np.abs(U - ex).max())
    if omega is not None:
        return errs
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(rates) > 1.8, (errs, rates)


def test_macro_laplacian_2d_equal_mode_exact():
    """closed form: for ω = (j, j) the one-point (rotated 5-point) operator's symbol
    4(s_x²c_y² + c_x²s_y²)/H² and the block-averaged exact load agree mode-wise, so the nodal values
    are exact to rounding (s = sin(θ/2), c = cos(θ/2), θ = jπH)."""
    errs = test_macro_laplacian_manufactured_rate(2, omega=[2, 2])
    assert max(errs) < 1e-12


def test_macro_operator_symmetric_and_decoupled():
    """a(U, V) = Σ_p t_p(V)ᵀ G_p t_p(U) is symmetric for symmetric G; with G block-diagonal in the
    continua (no coupling terms) the continua decouple exactly (SPEC structural-zero example)."""
    rng = np.random.default_rng(3)
    d, N, M = 2, 2, 6
    nr = N * (1 + d)
    G = np.zeros((M * M, nr, nr))
    for p in range(M * M):
        Q = rng.normal(size=(nr, nr))
        G[p] = Q @ Q.T
    K, F = block_operator(d, N, M, G, np.zeros((M * M, N)))
    assert abs(K - K.T).max() < 1e-12 * abs(K).max()
    mask = np.zeros((nr, nr), dtype=bool)
    idx = [[0, 2, 3], [1, 4, 5]]  # continuum 0: U_0, ∂U_0; continuum 1: U_1, ∂U_1
    for a in idx:
        mask[np.ix_(a, a)] = True
    K2, _ = block_operator(d, N, M, G * mask, np.zeros((M * M, N)))
    K2 = K2.toarray()
    assert np.abs(K2[0::2, 1::2]).max() == 0.0 and np.abs(K2[1::2, 0::2]).max() == 0.0
