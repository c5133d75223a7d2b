"""Oracle global fine solve and validation metrics (NEXT-3; TEST INFRASTRUCTURE ONLY — see
oracle/__init__.py).

* Fine-grid reference solution of Eq. (2): find u ∈ V_h ⊂ H¹₀(Ω), V_h = Q1 on
  the n^d fine cells, with ∫ κ ∇u·∇v = ∫ f v for all v ∈ V_h; u = 0 on ∂Ω (Eq. 1).
  κ and f cellwise constant; ∫_e f N_a = f_e h^d / 2^d (exact).  Assembled with
  ``fem.assemble_stiffness`` and solved by SciPy's sparse direct solver on the interior nodes.
* Fine block averages: ū_{p,i} = (1/|K_p ∩ Ω_i|) ∫_{K_p ∩ Ω_i} u, Ω_i the cells
  of continuum i; ∫_e u = h^d · (mean of the 2^d corner values) (exact for Q1).
* Macro block averages: (1/|K_p|) ∫_{K_p} U_i for U_i Q1 on the coarse vertex grid (block layout,
  K_p = block p) = mean of the block's 2^d corner values.
* Relative L² error e₂^{(i)} = sqrt(Σ_p |Ū_{p,i} − ū_{p,i}|² / Σ_p |ū_{p,i}|²).
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse.linalg as spla

from .fem import assemble_stiffness


def fine_load(f: np.ndarray) -> np.ndarray:
    """F_a = Σ_{cells e ∋ a} f_e h^d / 2^d, nodal array [.., y, x] of shape (n+1)^d."""
    d, n = f.ndim, f.shape[0]
    h = 1.0 / n
    F = np.zeros((n + 1,) * d)
    w = f * h ** d / 2 ** d
    for a in itertools.product((0, 1), repeat=d):
        sl = tuple(slice(ai, ai + n) for ai in a)
        F[sl] += w
    return F


def fine_solve(kappa: np.ndarray, f: np.ndarray) -> np.ndarray:
    """u nodal [.., y, x], (n+1)^d, zero on the boundary."""
    d, n = kappa.ndim, kappa.shape[0]
    h = 1.0 / n
    A = assemble_stiffness(np.asarray(kappa, dtype=np.float64), h).tocsr()
    F = fine_load(np.asarray(f, dtype=np.float64)).reshape(-1)
    interior = np.ones((n + 1,) * d, dtype=bool)
    for ax in range(d):
        idx = [slice(None)] * d
        idx[ax] = 0
        interior[tuple(idx)] = False
        idx[ax] = n
        interior[tuple(idx)] = False
    m = interior.reshape(-1)
    u = np.zeros((n + 1) ** d)
    u[m] = spla.spsolve(A[m][:, m].tocsc(), F[m])
    return u.reshape((n + 1,) * d)


def cell_means(u: np.ndarray) -> np.ndarray:
    """(1/|e|) ∫_e u for every fine cell: mean of the 2^d corner values."""
    d = u.ndim
    n = u.shape[0] - 1
    acc = np.zeros((n,) * d)
    for a in itertools.product((0, 1), repeat=d):
        acc += u[tuple(slice(ai, ai + n) for ai in a)]
    return acc / 2 ** d


def fine_block_averages(u: np.ndarray, ids: np.ndarray, N: int, M: int) -> np.ndarray:
    """ū[P][N] over the M^d blocks K_p (block layout, lexicographic x fastest)."""
    d = u.ndim
    n = u.shape[0] - 1
    c = n // M
    cm = cell_means(u)
    out = np.full((M ** d, N), np.nan)
    for kb in itertools.product(range(M), repeat=d):  # kb = (k_{d-1}, .., k_0)
        sl = tuple(slice(k * c, (k + 1) * c) for k in kb)
        p = sum(kb[d - 1 - i] * M ** i for i in range(d))
        for i in range(N):
            sel = ids[sl] == i
            if sel.any():
                out[p, i] = cm[sl][sel].mean()  # equal cell volumes: the mean of cell means
    return out


def macro_block_averages(U: np.ndarray, d: int, M: int) -> np.ndarray:
    """Ū[P][N] from nodal U[N][(M+1)^d] (block layout)."""
    N = U.shape[0]
    nv = M + 1
    out = np.zeros((M ** d, N))
    for p in range(M ** d):
        kb = [(p // M ** i) % M for i in range(d)]
        for a in range(2 ** d):
            node = sum((kb[i] + ((a >> i) & 1)) * nv ** i for i in range(d))
            out[p] += U[:, node]
    return out / 2 ** d


def e2(Ubar: np.ndarray, ubar: np.ndarray) -> np.ndarray:
    """e₂^{(i)} per continuum; macropoints where ū is undefined are skipped."""
    ok = np.isfinite(ubar)
    num = np.where(ok, (Ubar - ubar) ** 2, 0.0).sum(axis=0)
    den = np.where(ok, ubar ** 2, 0.0).sum(axis=0)
    return np.sqrt(num / den)
