"""Oracle saddle-point solve (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Solves   min ½ ξᵀAξ − bᵀξ   s.t.  Cξ = g
via the KKT system [[A, Cᵀ], [C, 0]] [ξ; λ] = [b; g]   (Eqs. 3-4 and 12-13 in
discrete form; the multipliers play the role of β).

Rows of C are equilibrated (each row divided by its measure ∫_{R_q}ψ_j and multiplied
by mean(diag A)), which leaves ξ unchanged; the sparse LU is SciPy's SuperLU with
MMD_AT_PLUS_A ordering, followed by one step of iterative refinement.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def solve_kkt(A: sp.spmatrix, C: sp.spmatrix, b: np.ndarray, g: np.ndarray,
              row_scale: np.ndarray | None = None, refine: int = 1):
    """A: n×n, C: m×n (full row rank), b: n×k, g: m×k.  Returns (ξ n×k, λ m×k, backward error)."""
    n = A.shape[0]
    m = C.shape[0]
    b = np.asarray(b, dtype=np.float64).reshape(n, -1)
    g = np.asarray(g, dtype=np.float64).reshape(m, -1)
    if row_scale is None:
        row_scale = np.ones(m)
    Dm = sp.diags(row_scale)
    Cs = (Dm @ C).tocsr()
    K = sp.bmat([[A, Cs.T], [Cs, None]], format="csc")
    rhs = np.vstack([b, row_scale[:, None] * g])
    lu = spla.splu(K, permc_spec="MMD_AT_PLUS_A")
    sol = lu.solve(rhs)
    for _ in range(refine):
        sol = sol + lu.solve(rhs - K @ sol)
    res = rhs - K @ sol
    kn = spla.norm(K, np.inf)
    berr = float(np.max(np.abs(res)) / (kn * max(np.max(np.abs(sol)), 1e-300) + np.max(np.abs(rhs)) + 1e-300))
    xi = sol[:n]
    lam = sol[n:] * row_scale[:, None]
    return xi, lam, berr
