"""Oracle upscaled system (NEXT-2; TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Load vectors (Eq. 7, PAPER.md:221 — b_j = |K_p|/|R_p| ∫_{R_p} f φ_j, with R_p = K_p,
PAPER.md:532, prefactor 1, reading R12), for a cellwise-constant source f:

    b_j(p) = Σ_{e ⊂ K_p} f_e ∫_e φ_j = Σ_{e ⊂ K_p} f_e (h^d / 2^d) Σ_{corners a of e} φ_j(a)

(exact: φ_j is Q1 on the fine grid, ∫_e N_a = h^d/2^d).

Macro system (Eq. 6 through the displayed bilinear form; "U_i, V_j and
their gradients are taken at specific points, such as the midpoint of the coarse block"),
on the block-centred layout (K_p = block p of side H): U_i continuous Q1 on the coarse vertex
grid {0..M}^d, homogeneous Dirichlet on ∂Ω ("u = 0 on ∂Ω", Eq. 1). With
t_p(U) = (U_0, .., U_{N-1}, ∂_0U_0, .., ∂_{d-1}U_0, .., ∂_{d-1}U_{N-1}) at the block centre
(the bilinear interpolant's value and gradient there; Gram order of Φ):

    a(U, V) = Σ_p t_p(V)ᵀ G_p t_p(U)        (G_p[a][b] = ∫_{K_p} κ ∇Φ_a·∇Φ_b, Eq. 7;
                                              U_iV_jB_ji, ∂_mU_iV_jB^m_ji, U_i∂_nV_jB̄^n_ji,
                                              ∂_mU_i∂_nV_jB^{mn}_ji term by term)
    l(V)    = Σ_p Σ_j V_j(x_p) b_j(p)

assembled explicitly (sparse) and solved by SciPy's direct sparse solver.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def load_vectors(oracle, f):
    """b[P][N] for every macropoint (block layout or vertex layout alike: over K_p)."""
    d, N, n, h = oracle.d, oracle.N, oracle.n, oracle.h
    f = np.asarray(f, dtype=np.float64).reshape((n,) * d)
    plan = oracle.plan
    out = np.zeros((plan.num_macropoints(), N))
    for k in plan.all_vertices():
        r = oracle.solve(k)
        lo, hi = r["lo"], r["hi"]
        c = plan.c
        # K_p fine-cell box (global), clipped to the window
        sub_lo = [max(lo[i], _kp_lo(plan, k[i])) for i in range(d)]
        sub_hi = [min(hi[i], _kp_lo(plan, k[i]) + c) for i in range(d)]
        phi = r["phi"]  # [rhs][nodes (z, y, x)]
        for j in range(N):
            acc = 0.0
            for e in itertools.product(*[range(sub_lo[i], sub_hi[i]) for i in range(d)]):
                fe = f[tuple(reversed(e))]
                s = 0.0
                for a in range(2 ** d):
                    node = tuple(e[i] - lo[i] + ((a >> i) & 1) for i in range(d))
                    s += phi[(j,) + tuple(reversed(node))]
                acc += fe * s * h ** d / 2 ** d
            out[plan.linear_index(k), j] = acc
    return out


def _kp_lo(plan, ki):
    """first fine cell of K_p along one dimension (K_p = the subcell of slot l)"""
    return ki * plan.c - (plan.c // 2 if plan.layout == "vertex" else 0)


def block_operator(d, N, M, G, b):
    """Sparse K, F over all (M+1)^d coarse nodes × N continua (node-major, continuum fastest),
    from per-block Gram matrices G[P][n_rhs][n_rhs] and loads b[P][N] (block layout)."""
    H = 1.0 / M
    nv = M + 1
    nr = N * (1 + d)
    rows, cols, vals = [], [], []
    F = np.zeros(nv ** d * N)
    for kb in itertools.product(range(M), repeat=d):
        kb = tuple(reversed(kb))  # x fastest ordering of blocks
        p = sum(kb[i] * M ** i for i in range(d))
        corners = [tuple(kb[i] + ((a >> i) & 1) for i in range(d)) for a in range(2 ** d)]
        cidx = [sum(c[i] * nv ** i for i in range(d)) for c in corners]
        # E: t_p = E @ u_local, u_local[a*N + i] = U_i(corner a)
        E = np.zeros((nr, 2 ** d * N))
        for a in range(2 ** d):
            for i in range(N):
                E[i, a * N + i] = 1.0 / 2 ** d
                for m in range(d):
                    sgn = 1.0 if (a >> m) & 1 else -1.0
                    E[N + i * d + m, a * N + i] = sgn / (H * 2 ** (d - 1))
        Ke = E.T @ G[p] @ E
        Fe = np.zeros(2 ** d * N)
        for a in range(2 ** d):
            for j in range(N):
                Fe[a * N + j] = b[p, j] / 2 ** d
        gi = [cidx[a] * N + i for a in range(2 ** d) for i in range(N)]
        for r_, gr in enumerate(gi):
            F[gr] += Fe[r_]
            for c_, gc in enumerate(gi):
                rows.append(gr)
                cols.append(gc)
                vals.append(Ke[r_, c_])
    K = sp.csr_matrix((vals, (rows, cols)), shape=(nv ** d * N, nv ** d * N))
    return K, F


def macro_solve(d, N, M, G, b):
    """U[N][(M+1)^d] nodal values (Dirichlet zeros on ∂Ω)."""
    nv = M + 1
    K, F = block_operator(d, N, M, G, b)
    interior = np.array([all(0 < ((node // nv ** i) % nv) < M for i in range(d))
                         for node in range(nv ** d)])
    free = np.repeat(interior, N)
    U = np.zeros(nv ** d * N)
    Kf = K[free][:, free].tocsc()
    U[free] = spla.spsolve(Kf, F[free])
    return U.reshape(nv ** d, N).T.copy()
