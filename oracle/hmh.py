"""Oracle driver for Algorithm 1 (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

For each level n = 1..L and each macropoint p ∈ S_n (Alg. 1 lines 3-7):

1. Window R_p^+ and subcells R_q (reading R2), fine assembly of A₁ (natural BC,
   reading R3) and of the constraint rows C₁ with measures ∫_{R_q}ψ_j; rows of
   zero measure are dropped (reading R13).
2. Centring constants c_mj: ∫_{K_p}(x_m − c_mj)ψ_j = 0, used in the
   targets of every R_q (reading R8).
3. Targets g⁰: avg type δ_ij∫_{R_q}ψ_j (Eq. 3); gradient type
   δ_ij∫_{R_q}(x_m − c_mj)ψ_j (Eq. 4).
4. Level space V_n on mesh hη^{n-1}: P_n explicit, A_n = P_nᵀA₁P_n,
   C_n = C₁P_n (exact Galerkin, reading R11).
5. n ≥ 2: I_p = Σ_t c_t φ_t(x_t + ·) (Eq. 11; readings R9/R10);
   b = −P_nᵀA₁I_p (first lines of Eqs. 12/13 with reading R5),
   g = g⁰ − C₁I_p (second lines of Eqs. 12/13).
   n = 1: I_p = 0.
6. KKT solve (oracle/kkt.py), φ_p = P_nξ + I_p (Eq. 11).
7. Gram G_p[a][b] = ∫_{K_p} κ∇Φ_a·∇Φ_b (Eq. 7, with R_p = K_p,
   PAPER.md:532, prefactor |K_p|/|R_p| = 1; reading R12), Φ ordered
   (φ_0..φ_{N-1}, φ_0^0..φ_0^{d-1}, .., φ_{N-1}^{d-1}) — B_ji = G[j][i],
   B^m_ji = G[j][N+i·d+m], B̄^n_ji = G[N+j·d+n][i], B^{mn}_ji = G[N+j·d+n][N+i·d+m].
"""
from __future__ import annotations

import os
import time

import numpy as np

from .fem import assemble_constraints, assemble_stiffness, prolongation
from .kkt import solve_kkt
from .planner import Plan


class OracleError(RuntimeError):
    pass


RANK_TOL = 1e-11


def constraint_rows(An, Cn, g):
    """Reading R20: if the level-n constraint rows are linearly dependent
    (the level mesh cannot separate the continua inside a subcell, i.e. PAPER.md:374's
    assumption that ηᴸ⁻¹h resolves the heterogeneity fails), the constraints are imposed in
    the least-squares sense for rows normalised in the D⁻¹ norm, D = diag(A_n):
    with S̃ = Λ C D⁻¹ Cᵀ Λ, Λ = diag(C D⁻¹ Cᵀ)^(-1/2), S̃ = V diag(λ) Vᵀ, keep the
    eigenvectors with λ > RANK_TOL·λ_max and replace (C, g) by (V_kᵀ Λ C, V_kᵀ Λ g).
    Full-rank systems are returned unchanged.  Returns (C, g, rank_deficient)."""
    import scipy.sparse as sp
    dinv = 1.0 / An.diagonal()
    S = (Cn @ sp.diags(dinv) @ Cn.T).toarray()
    lam = 1.0 / np.sqrt(np.diag(S))
    St = S * lam[:, None] * lam[None, :]
    ev, V = np.linalg.eigh(St)
    keep = ev > RANK_TOL * ev.max()
    if keep.all():
        return Cn, g, False
    Vk = V[:, keep]
    Cr = sp.csr_matrix(Vk.T @ (lam[:, None] * Cn.toarray()))
    gr = Vk.T @ (lam[:, None] * g)
    return Cr, gr, True


class Oracle:
    def __init__(self, d, n, M, L, eta, N, kappa, ids, l=1, keep_all_phi=False, interp="dlinear",
                 layout="vertex"):
        self.plan = Plan(d, n, M, L, eta, l, interp=interp, layout=layout)
        self.d, self.n, self.M, self.L, self.eta, self.N, self.l = d, n, M, L, eta, N, l
        self.h = 1.0 / n
        self.kappa = np.asarray(kappa, dtype=np.float64).reshape((n,) * d)
        self.ids = np.asarray(ids, dtype=np.uint8).reshape((n,) * d)
        if np.any(self.ids >= N):
            raise OracleError("continuum id >= N")
        self.n_rhs = N * (1 + d)
        self.keep_all_phi = keep_all_phi
        self.cache = {}
        self.timings = {}

    @classmethod
    def from_config(cls, cfg, kappa, ids, **kw):
        return cls(cfg.d, cfg.n, cfg.M, cfg.L, cfg.eta, cfg.N, kappa, ids, l=cfg.l, **kw)

    # ------------------------------------------------------------------------
    def _slices(self, lo, hi):
        return tuple(slice(lo[i], hi[i]) for i in reversed(range(self.d)))

    def _axis_shape(self, i, length):
        sh = [1] * self.d
        sh[self.d - 1 - i] = length
        return sh

    def local_system(self, k):
        """Everything of steps 1-4 for macropoint k (also used by tests)."""
        d, N, h, c = self.d, self.N, self.h, self.plan.c
        l = self.plan.l_of(k)
        lev = self.plan.level_of(k)
        lo, hi = self.plan.window(k)
        sl = self._slices(lo, hi)
        kap = self.kappa[sl]
        idb = self.ids[sl]
        cells = tuple(hi[i] - lo[i] for i in range(d))
        w = 2 * l + 1
        sub = np.zeros(kap.shape, dtype=np.int64)
        for i in range(d):
            gi = np.arange(lo[i], hi[i])
            slot = self.plan.subcell_coord(gi) - k[i] + l
            sub = sub + (slot * w ** i).reshape(self._axis_shape(i, len(gi)))
        n_sub = w ** d
        A1 = assemble_stiffness(kap, h)
        C1, V = assemble_constraints(idb, sub, n_sub, N, h)
        active = V > 0
        cen = self.plan.centre_subcell(k)
        # centring constants on K_p
        cm = np.zeros((d, N))
        xc = [((np.arange(lo[i], hi[i]) + 0.5) * h).reshape(self._axis_shape(i, hi[i] - lo[i]))
              for i in range(d)]
        for j in range(N):
            mask = (sub == cen) & (idb == j)
            cnt = int(mask.sum())
            if cnt == 0:
                raise OracleError(f"continuum {j} absent from K_p of macropoint {k}")
            for m in range(d):
                cm[m, j] = np.broadcast_to(xc[m], kap.shape)[mask].sum() / cnt
        # targets g0 (rows q*N+j, columns rhs)
        row_e = (sub * N + idb).reshape(-1)
        g0 = np.zeros((n_sub * N, self.n_rhs))
        for j in range(N):
            rows = np.arange(n_sub) * N + j
            g0[rows, j] = V[rows]
            for m in range(d):
                xm = np.broadcast_to(xc[m], kap.shape).reshape(-1)
                sel = idb.reshape(-1) == j
                sx = np.bincount(row_e[sel], weights=xm[sel], minlength=n_sub * N)
                cnt = np.bincount(row_e[sel], minlength=n_sub * N).astype(np.float64)
                g0[rows, N + j * d + m] = h ** d * (sx[rows] - cm[m, j] * cnt[rows])
        s = self.eta ** (lev - 1)
        P = prolongation(cells, s)
        return dict(level=lev, lo=lo, hi=hi, cells=cells, kap=kap, ids=idb, sub=sub, A1=A1, C1=C1,
                    V=V, active=active, cm=cm, g0=g0, P=P, cen=cen)

    def transport(self, k, lo, hi):
        """I_p on the child's fine window nodes, shape (n_rhs, nodes) (Eq. 11, reading R9)."""
        d, c = self.d, self.plan.c
        nodes_shape = tuple(hi[i] - lo[i] + 1 for i in reversed(range(d)))
        I = np.zeros((self.n_rhs,) + nodes_shape)
        for t, wt in self.plan.parents(k):
            pt = self.solve(t)
            src = []
            for i in reversed(range(d)):
                # local coordinates (R9): shift by x_t - x_p; physical (NEXT-4): none
                shift = 0 if self.plan.interp == "physical_s1" else (t[i] - k[i]) * c
                a = lo[i] + shift - pt["lo"][i]
                src.append(slice(a, a + hi[i] - lo[i] + 1))
            I += wt * pt["phi"][(slice(None),) + tuple(src)]
        return I.reshape(self.n_rhs, -1)

    def solve(self, k):
        k = tuple(int(v) for v in k)
        if k in self.cache:
            return self.cache[k]
        t0 = time.perf_counter()
        S = self.local_system(k)
        A1, C1, P, active = S["A1"], S["C1"], S["P"], S["active"]
        An = (P.T @ A1 @ P).tocsr()
        Cn = (C1 @ P).tocsr()
        if S["level"] >= 2:
            I = self.transport(k, S["lo"], S["hi"])
            b = -(P.T @ (A1 @ I.T))
            g = S["g0"] - C1 @ I.T
        else:
            I = None
            b = np.zeros((An.shape[0], self.n_rhs))
            g = S["g0"]
        Ca, ga, rank_def = constraint_rows(An, Cn[active], g[active])
        if rank_def:
            scale = np.full(Ca.shape[0], float(np.mean(An.diagonal())) / np.abs(Ca).sum(axis=1).max())
        else:
            scale = float(np.mean(An.diagonal())) / S["V"][active]
        xi, lam, berr = solve_kkt(An, Ca, b, ga, row_scale=scale)
        phi = (P @ xi).T
        if I is not None:
            phi = phi + I
        Akp = assemble_stiffness(S["kap"], self.h, mask=(S["sub"] == S["cen"]))
        G = phi @ (Akp @ phi.T)
        nodes_shape = tuple(S["hi"][i] - S["lo"][i] + 1 for i in reversed(range(self.d)))
        res = dict(level=S["level"], lo=S["lo"], hi=S["hi"], G=G, berr=berr,
                   phi=phi.reshape((self.n_rhs,) + nodes_shape), xi=xi, cm=S["cm"])
        self.cache[k] = res
        self.timings[k] = time.perf_counter() - t0
        return res

    # ------------------------------------------------------------------------
    def run(self, points=None):
        """Solve all macropoints (levels in order) or the given subset (plus the parents it
        needs).  Returns {k: G}."""
        if points is None:
            points = [k for lev in range(1, self.L + 1) for k in self.plan.S(lev)]
        return {tuple(k): self.solve(k)["G"] for k in points}

    def effective_coeffs(self):
        """G for all (M+1)^d macropoints in lexicographic order, shape [P, n_rhs, n_rhs]."""
        out = np.zeros((self.plan.num_macropoints(), self.n_rhs, self.n_rhs))
        for lev in range(1, self.L + 1):
            for k in self.plan.S(lev):
                out[self.plan.linear_index(k)] = self.solve(k)["G"]
        return out


# -- process-pool timing helper (cpu_baseline / --impl reference) ---------------
_POOL_ORACLE = None


_POOL_KEEP = False


def _pool_solve(k):
    r = _POOL_ORACLE.solve(k)
    keep = _POOL_KEEP or r["level"] < _POOL_ORACLE.L
    return k, r["G"], (r["phi"] if keep else None), _POOL_ORACLE.timings[k]


def run_parallel(oracle: Oracle, points_by_level, workers=None, keep_phi=False):
    """Solve macropoints level by level with a fork-based process pool (one macropoint
    per task); parents must be in earlier levels of ``points_by_level``.  Returns
    (per-level wall seconds, workers used)."""
    import multiprocessing as mp
    global _POOL_ORACLE, _POOL_KEEP
    _POOL_KEEP = keep_phi
    workers = workers or len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    walls = []
    for pts in points_by_level:
        _POOL_ORACLE = oracle
        t0 = time.perf_counter()
        if workers == 1 or len(pts) <= 1:
            for k in pts:
                oracle.solve(k)
        else:
            with ctx.Pool(min(workers, len(pts))) as pool:
                for k, G, phi, tt in pool.imap_unordered(_pool_solve, [tuple(p) for p in pts]):
                    oracle.cache[k] = dict(level=oracle.plan.level_of(k), G=G, phi=phi,
                                           lo=oracle.plan.window(k)[0], hi=oracle.plan.window(k)[1])
                    oracle.timings[k] = tt
        walls.append(time.perf_counter() - t0)
    return walls, workers
