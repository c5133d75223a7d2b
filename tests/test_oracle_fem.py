"""Pins for oracle/fem.py and oracle/kkt.py."""
import itertools

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.fem import (assemble_constraints, assemble_stiffness, prolongation, prolongation_1d,
                        q1_element_stiffness)
from oracle.kkt import solve_kkt


def test_q1_2d_textbook():
    """Unit-square bilinear element: diagonal 2/3, edge neighbours −1/6, opposite corner −1/3
    (textbook).  Corner order (0,0),(1,0),(0,1),(1,1)."""
    want = np.array([[4, -1, -1, -2], [-1, 4, -2, -1], [-1, -2, 4, -1], [-2, -1, -1, 4]]) / 6.0
    for h in (1.0, 0.125):
        assert np.allclose(q1_element_stiffness(2, h), want, atol=1e-15, rtol=0)  # h^{d-2} = 1


def test_q1_3d_textbook():
    """Unit-cube trilinear element: diagonal 1/3, edge neighbours 0, face and body diagonals
    −1/12, scaled by h^{d-2} = h."""
    h = 0.25
    K = q1_element_stiffness(3, h)
    for a, b in itertools.product(range(8), repeat=2):
        nd = bin(a ^ b).count("1")
        want = {0: 1 / 3, 1: 0.0, 2: -1 / 12, 3: -1 / 12}[nd] * h
        assert abs(K[a, b] - want) < 1e-15


@pytest.mark.parametrize("d", [2, 3])
def test_q1_gauss_quadrature(d):
    """Element stiffness equals 2-point Gauss quadrature of ∇N_a·∇N_b (exact for Q1)."""
    h = 0.3
    gp = np.array([0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)])
    K = np.zeros((2 ** d, 2 ** d))
    for pt in itertools.product(gp, repeat=d):
        grads = []
        for a in range(2 ** d):
            g = []
            for k in range(d):
                v = 1.0
                for i in range(d):
                    ai = (a >> i) & 1
                    if i == k:
                        v *= (1.0 if ai else -1.0) / h
                    else:
                        v *= pt[i] if ai else 1 - pt[i]
                g.append(v)
            grads.append(np.array(g))
        w = (0.5 * h) ** d
        for a in range(2 ** d):
            for b in range(2 ** d):
                K[a, b] += w * grads[a] @ grads[b]
    assert np.allclose(q1_element_stiffness(d, h), K, atol=1e-13)


@pytest.mark.parametrize("d", [2, 3])
def test_assembly_constants_and_dense(d):
    rng = np.random.default_rng(0)
    shape = (3, 4, 5)[:d]
    kap = rng.uniform(1, 10, shape)
    h = 0.1
    A = assemble_stiffness(kap, h).toarray()
    assert np.abs(A @ np.ones(A.shape[0])).max() < 1e-12
    assert np.abs(A - A.T).max() < 1e-15
    # dense per-element summation with explicit index arithmetic
    nn = [s + 1 for s in reversed(shape)]
    Ke = q1_element_stiffness(d, h)
    B = np.zeros_like(A)
    for e in itertools.product(*[range(s) for s in reversed(shape)]):  # e = (ex, ey[, ez])
        nodes = []
        for a in range(2 ** d):
            idx = 0
            for i in reversed(range(d)):
                idx = idx * nn[i] + e[i] + ((a >> i) & 1)
            nodes.append(idx)
        B[np.ix_(nodes, nodes)] += kap[tuple(reversed(e))] * Ke
    assert np.allclose(A, B, atol=1e-12)


def test_constraint_row_sums_are_measures():
    """C·1 = ∫_{R_q}ψ_j."""
    rng = np.random.default_rng(1)
    ids = rng.integers(0, 3, (6, 6)).astype(np.uint8)
    sub = np.zeros((6, 6), dtype=np.int64)
    sub[:, 3:] = 1
    h = 0.5
    C, V = assemble_constraints(ids, sub, 2, 3, h)
    assert np.allclose(C @ np.ones(C.shape[1]), V)
    for q in range(2):
        for j in range(3):
            assert V[q * 3 + j] == h * h * np.sum((sub == q) & (ids == j))


def test_prolongation_constants_linears_composition():
    P = prolongation((8, 4), 2)
    xc = np.arange(5) * 2.0
    yc = np.arange(3) * 2.0
    Xc, Yc = np.meshgrid(xc, yc)
    Xf, Yf = np.meshgrid(np.arange(9.0), np.arange(5.0))
    assert np.allclose(P @ np.ones(P.shape[1]), 1.0)
    assert np.allclose(P @ Xc.reshape(-1), Xf.reshape(-1))
    assert np.allclose(P @ Yc.reshape(-1), Yf.reshape(-1))
    # η=2 twice equals η=4
    P4 = prolongation_1d(2, 4).toarray()
    P22 = prolongation_1d(4, 2).toarray() @ prolongation_1d(2, 2).toarray()
    assert np.allclose(P4, P22, atol=1e-15)


def test_kkt_1d_hand_solve():
    """A=[[2]], C=[[1]], b=0, g=3 → ξ=3; 2·3 + λ = 0 → λ = −6."""
    import scipy.sparse as sp
    xi, lam, _ = solve_kkt(sp.csr_matrix([[2.0]]), sp.csr_matrix([[1.0]]), np.zeros(1), np.array([3.0]))
    assert abs(xi[0, 0] - 3.0) < 1e-14 and abs(lam[0, 0] + 6.0) < 1e-14


def test_kkt_vs_nullspace_method():
    """Random semidefinite A (constant null space) + constraints, ≤ 200 unknowns: sparse KKT LU
    equals the null-space method ξ = ξ_p + Z y (a different algorithm)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(2)
    kap = rng.uniform(1, 100, (9, 9))
    A = assemble_stiffness(kap, 0.1)
    n = A.shape[0]
    C = sp.csr_matrix(rng.uniform(0, 1, (7, n)) * (rng.uniform(0, 1, (7, n)) < 0.3))
    b = rng.standard_normal((n, 2))
    b -= b.mean(axis=0)
    g = rng.standard_normal((7, 2))
    xi, lam, berr = solve_kkt(A, C, b, g)
    Cd, Ad = C.toarray(), A.toarray()
    xp = np.linalg.lstsq(Cd, g, rcond=None)[0]
    Z = sla.null_space(Cd)
    y = np.linalg.solve(Z.T @ Ad @ Z, Z.T @ (b - Ad @ xp))
    ref = xp + Z @ y
    assert np.abs(xi - ref).max() / np.abs(ref).max() < 1e-10
    assert berr < 1e-13
