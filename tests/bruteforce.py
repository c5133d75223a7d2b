"""Dense brute-force implementation of the hierarchical cell problems for tiny grids.

Independent of oracle/ (imports nothing from it): every integral is computed by
2-point Gauss quadrature from explicit multilinear basis formulas, the level-n
space by evaluating coarse hat functions at fine nodes, parents by enumerating
T_{n-1}, and the constrained minimum by the null-space method (SVD of C), not a
KKT factorisation.  Pins oracle/hmh.py.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.linalg as sla

GP = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])


def _vertices(d, M):
    return [tuple(reversed(r)) for r in itertools.product(range(M + 1), repeat=d)]


class BruteForce:
    def __init__(self, d, n, M, L, eta, N, kappa, ids, l=1, layout="vertex", physical=False):
        self.d, self.n, self.M, self.L, self.eta, self.N, self.l = d, n, M, L, eta, N, l
        self.layout = layout
        # NEXT-4: nearest S_1 parent in physical coordinates, level-1 regions
        # enlarged to contain the windows of every child assigned to them
        self.physical = physical
        self.h = 1.0 / n
        self.H = 1.0 / M
        self.kappa = kappa.reshape((n,) * d)
        self.ids = ids.reshape((n,) * d)
        self.n_rhs = N * (1 + d)
        self.res = {}
        if layout == "block":
            self._block_levels()

    def points(self):
        m = self.M + 1 if self.layout == "vertex" else self.M
        return [tuple(reversed(r)) for r in itertools.product(range(m), repeat=self.d)]

    def xp(self, k):
        off = 0.5 if self.layout == "block" else 0.0
        return [(ki + off) * self.H for ki in k]

    def _block_levels(self):
        """T_n of the block layout by enumerating coarse blocks in physical space: T_L = every
        block; each coarse block of size η^{L-n}H keeps the T_{n+1} point inside it whose centre is
        closest to the block's centre (ties: the smaller coordinates)."""
        self.Tsets = {self.L: set(self.points())}
        for lev in range(self.L - 1, 0, -1):
            S = self.eta ** (self.L - lev) * self.H
            nb = int(round(1.0 / S))
            keep = set()
            for cb in itertools.product(range(nb), repeat=self.d):
                inside = [t for t in self.Tsets[lev + 1]
                          if all(cb[i] * S - 1e-12 <= self.xp(t)[i] < (cb[i] + 1) * S - 1e-12 for i in range(self.d))]
                centre = [(cb[i] + 0.5) * S for i in range(self.d)]
                best = min(inside, key=lambda t: (round(max(abs(self.xp(t)[i] - centre[i])
                                                            for i in range(self.d)) / self.H, 9),
                                                  tuple(reversed(t))))
                keep.add(best)
            self.Tsets[lev] = keep

    def in_T(self, k, lev):
        if self.layout == "block":
            return k in self.Tsets[lev]
        return all(ki % self.eta ** (self.L - lev) == 0 for ki in k)

    def level(self, k):
        for lev in range(1, self.L + 1):
            if self.in_T(k, lev):
                return lev

    def lk(self, k):
        """layers of k's window: level-1 points of the physical variant reach every assigned child,
        i.e. the children within half the S_1 spacing, η^{L-1}H/2"""
        if self.physical and self.level(k) == 1:
            return self.l + self.eta ** (self.L - 1) // 2
        return self.l

    def window(self, k):
        """physical box [a_i, b_i] of R_p^+ = x_p ± (l+1/2)H clipped to [0,1]"""
        r = (self.lk(k) + 0.5) * self.H
        return [(max(0.0, x - r), min(1.0, x + r)) for x in self.xp(k)]

    def parents(self, k):
        lev = self.level(k)
        if self.physical:  # the S_1 point nearest to x_p (max-norm ties: smaller coordinates)
            S1 = [t for t in self.points() if self.level(t) == 1]
            best = min(S1, key=lambda t: (sum((t[i] - k[i]) ** 2 for i in range(self.d)), tuple(reversed(t))))
            return [(best, 1.0)]
        s = self.eta ** (self.L - lev + 1)
        Tprev = [t for t in self.points() if self.in_T(t, lev - 1)]
        # per coordinate: candidate lattice values within distance < s, linear weights
        per = []
        wk = self.window(k)
        for i, ki in enumerate(k):
            cands = sorted({t[i] for t in Tprev if abs(t[i] - ki) < s})
            ws = {ti: 1.0 - abs(ti - ki) / s for ti in cands}
            ok = []
            for ti in cands:
                tw = self.window(tuple(ti if j == i else k[j] for j in range(self.d)))[i]
                # parent window, shifted to the child's centre, must contain the child's window
                sh = (ki - ti) * self.H
                if tw[0] + sh <= wk[i][0] + 1e-12 and tw[1] + sh >= wk[i][1] - 1e-12:
                    ok.append(ti)
            if len(ok) < len(cands):
                ws = {ok[0]: 1.0}
            tot = sum(ws[ti] for ti in ok)  # Σ c_t = 1 with one-sided neighbours
            per.append([(ti, ws[ti] / tot) for ti in ok])
        out = []
        for combo in itertools.product(*per):
            out.append((tuple(c[0] for c in combo), float(np.prod([c[1] for c in combo]))))
        return out

    def solve(self, k):
        if k in self.res:
            return self.res[k]
        d, h, N = self.d, self.h, self.N
        lev = self.level(k)
        box = self.window(k)
        ncell = [int(round((b - a) / h)) for a, b in box]
        x0 = [a for a, _ in box]
        nodes = list(itertools.product(*[range(c + 1) for c in reversed(ncell)]))  # (z,y,x) order
        nodes = [tuple(reversed(nd)) for nd in nodes]  # (x,y,z), x fastest in list order
        nid = {nd: i for i, nd in enumerate(nodes)}
        X = np.array([[x0[i] + nd[i] * h for i in range(d)] for nd in nodes])
        nn = len(nodes)
        # coarse nodes of V_n: spacing hc = h*eta^(lev-1)
        hc = h * self.eta ** (lev - 1)
        ncc = [c // self.eta ** (lev - 1) for c in ncell]
        cnodes = [tuple(reversed(r)) for r in itertools.product(*[range(c + 1) for c in reversed(ncc)])]
        Y = np.array([[x0[i] + cn[i] * hc for i in range(d)] for cn in cnodes])
        P = np.ones((nn, len(cnodes)))
        for i in range(d):
            P *= np.maximum(0.0, 1.0 - np.abs(X[:, i:i + 1] - Y[None, :, i]) / hc)
        # quadrature over fine elements
        A1 = np.zeros((nn, nn))
        AK = np.zeros((nn, nn))
        lk = self.lk(k)
        nsub = (2 * lk + 1) ** d
        C1 = np.zeros((nsub * N, nn))
        V = np.zeros(nsub * N)
        mom = np.zeros((nsub * N, d))     # ∫_{R_q} x_m ψ_j
        kmom = np.zeros((N, d + 1))       # ∫_{K_p} ψ_j, ∫_{K_p} x_m ψ_j
        # reference-element quadrature tables (same for every fine element: uniform h)
        qN, qG, qW, qX = [], [], [], []
        for pt in itertools.product(GP, repeat=d):
            Nv = np.ones(2 ** d)
            grad = np.ones((2 ** d, d))
            for a in range(2 ** d):
                for i in range(d):
                    ai = (a >> i) & 1
                    Nv[a] *= pt[i] if ai else 1 - pt[i]
                    for m in range(d):
                        if m == i:
                            grad[a, m] *= (1.0 if ai else -1.0) / h
                        else:
                            grad[a, m] *= pt[i] if ai else 1 - pt[i]
            qN.append(Nv); qG.append(grad); qW.append(h ** d / 2 ** d); qX.append(np.array(pt))
        Kref = sum(w * g @ g.T for w, g in zip(qW, qG))
        Mvec = sum(w * nv for w, nv in zip(qW, qN))
        for e in itertools.product(*[range(c) for c in ncell]):
            corner = [tuple(e[i] + ((a >> i) & 1) for i in range(d)) for a in range(2 ** d)]
            cid = [nid[c] for c in corner]
            gcell = tuple(int(round(x0[i] / h)) + e[i] for i in range(d))
            kap = self.kappa[tuple(reversed(gcell))]
            j = int(self.ids[tuple(reversed(gcell))])
            centre = [x0[i] + (e[i] + 0.5) * h for i in range(d)]
            vq = [int(np.floor(centre[i] / self.H + (0.5 if self.layout == "vertex" else 0.0)))
                  for i in range(d)]
            q = 0
            for i in reversed(range(d)):
                q = q * (2 * lk + 1) + (vq[i] - k[i] + lk)
            in_kp = all(vq[i] == k[i] for i in range(d))
            Ke = kap * Kref
            A1[np.ix_(cid, cid)] += Ke
            xm = sum(w * (np.array(x0) + (np.array(e) + xq) * h) for w, xq in zip(qW, qX))
            vol = sum(qW)
            if in_kp:
                AK[np.ix_(cid, cid)] += Ke
                kmom[j, 0] += vol
                kmom[j, 1:] += xm
            C1[q * N + j, cid] += Mvec
            V[q * N + j] += vol
            mom[q * N + j] += xm
        cm = kmom[:, 1:] / kmom[:, :1]  # (N, d) centroid of continuum j in K_p
        g0 = np.zeros((nsub * N, self.n_rhs))
        for q in range(nsub):
            for j in range(N):
                r = q * N + j
                g0[r, j] = V[r]
                for m in range(d):
                    g0[r, N + j * d + m] = mom[r, m] - cm[j, m] * V[r]
        active = V > 1e-300
        I = np.zeros((nn, self.n_rhs))
        if lev >= 2:
            for t, w in self.parents(k):
                pt = self.solve(t)
                shift = np.zeros(d) if self.physical else np.array([(t[i] - k[i]) * self.H for i in range(d)])
                Xt = X + shift
                idx = [pt["nid"][tuple(int(round((Xt[a, i] - pt["x0"][i]) / h)) for i in range(d))]
                       for a in range(nn)]
                I += w * pt["phi"][idx]
        An = P.T @ A1 @ P
        Cn = (C1 @ P)[active]
        b = -P.T @ (A1 @ I)
        g = (g0 - C1 @ I)[active]
        # rows normalised in the D⁻¹ norm (D = diag A_n); constraints imposed in the
        # least-squares sense when the level-n rows are dependent (reading R20)
        dn = np.diag(An)
        ds = 1.0 / np.sqrt(np.einsum("ij,j,ij->i", Cn, 1.0 / dn, Cn))
        Cn = ds[:, None] * Cn
        g = ds[:, None] * g
        xp = np.linalg.lstsq(Cn, g, rcond=1e-9)[0]
        Z = sla.null_space(Cn, rcond=1e-9)
        y = np.linalg.solve(Z.T @ An @ Z, Z.T @ (b - An @ xp))
        xi = xp + Z @ y
        phi = P @ xi + I
        G = phi.T @ AK @ phi
        out = dict(phi=phi, nid=nid, x0=x0, G=G, C1=C1[active], g0=g0[active], A1=A1, level=lev,
                   nodes=nodes, ncell=ncell)
        self.res[k] = out
        return out
