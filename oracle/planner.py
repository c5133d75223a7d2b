"""Oracle macrogrid hierarchy (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Vertex-centred macrogrid (reading R1): macropoints x_p = H·k, k ∈ {0..M}^d,
K_p = R_p = Π[x_p,i ± H/2] ∩ Ω ("R_p = K_p").

* T_n = {k : k_i ≡ 0 mod η^{L-n}}  — nested grids of spacing η^{L-n}H
  (§3.1; reading R7).
* S_1 = T_1, S_n = T_n \\ ∪_{k<n} S_k = T_n \\ T_{n-1}  (Eq. 10).
* R_p^+ = Π[x_p,i ± (l+1/2)H] ∩ Ω, subcells R_q = dual blocks of the vertices
  with ‖x_q − x_p‖∞ ≤ lH (reading R2).
* Parents of p ∈ S_n (n ≥ 2): the corners of the T_{n-1} cell containing x_p with
  d-linear weights Π_i (1 − |x_p,i − x_t,i| / s_{n-1}), Σ c_t = 1 (Eq. 11,
  PAPER.md:382-389; reading R10).  A parent whose window does not cover the
  child's (local-coordinate transport, reading R9) is dropped per coordinate and
  its weight given to the opposite parent.

Block-centred layout (NEXT-1, the paper's own figures, Figs. 2-3): macropoints
at block centres x_p = (k + ½)H, k ∈ {0..M−1}^d, K_p = the block, R_p^+ = K_p ± lH, subcells =
the blocks of R_p^+.  T_n = {k : k_i ≡ r_n mod η^{L-n}}: each coarse block of size η^{L-n}H keeps
one macropoint, the finest block of T_{n+1} inside it whose centre is closest
to the coarse block's centre (ties: the smaller index) — r_L = 0, which reproduces Fig. 2
(H = 1/8, η = 2: T_1 at blocks {2, 6}, T_2 at {0, 2, 4, 6}).  Parents: d-linear on the T_{n-1}
lattice where x_p lies between two lattice points, the single nearer-side point otherwise; then
the R9 covering rule as above.

Lexicographic order: x (k[0]) fastest.
"""
from __future__ import annotations

import itertools
import math


def oversampling_layers_paper(H: float) -> int:
    """l = ⌈−2 log H⌉ with the natural log (§4; Table 1 prints 5, 7, 8
    for H = 1/12, 1/24, 1/48)."""
    return int(math.ceil(-2.0 * math.log(H) - 1e-12))


def block_offsets(L: int, eta: int):
    """r_n (n = 1..L) of the block-centred hierarchy: r_L = 0; r_n is the T_{n+1} block inside the
    coarse block [0, η^{L-n}) whose centre is closest to the coarse centre (ties: smaller)."""
    r = {L: 0}
    for lev in range(L - 1, 0, -1):
        s, s1 = eta ** (L - lev), eta ** (L - lev - 1)
        cands = [r[lev + 1] + j * s1 for j in range(eta)]
        r[lev] = min(cands, key=lambda v: (abs(v + 0.5 - s / 2), v))
    return r


class Plan:
    def __init__(self, d: int, n: int, M: int, L: int, eta: int, l: int = 1, interp: str = "dlinear",
                 layout: str = "vertex"):
        if n % M:
            raise ValueError("M must divide n (H/h integer)")
        self.d, self.n, self.M, self.L, self.eta, self.l = d, n, M, L, eta, l
        if interp not in ("dlinear", "nearest_s1", "physical_s1"):
            raise ValueError("interp must be 'dlinear', 'nearest_s1' or 'physical_s1'")
        if interp == "physical_s1" and layout != "vertex":
            raise ValueError("the physical-coordinate variant is built for the vertex layout")
        if layout not in ("vertex", "block"):
            raise ValueError("layout must be 'vertex' or 'block'")
        self.interp, self.layout = interp, layout
        self.c = n // M  # fine cells per H
        # both layouts: H/(2h) and H/(2 h η^{L-1}) integers, i.e. the coarsest level mesh has at
        # least two elements across every subcell (PAPER.md:374 assumes η^{L-1}h resolves the
        # heterogeneity; with one element per subcell the constraint rows are dependent everywhere)
        if self.c % 2:
            raise ValueError("H/(2h) must be an integer")
        if (self.c // 2) % (eta ** (L - 1)):
            raise ValueError("H/(2 h eta^(L-1)) must be an integer")
        if M % (eta ** (L - 1)):
            raise ValueError("eta^(L-1) must divide M")
        # macropoint coordinates per dimension, fine-cell position of x_p (doubled to stay
        # integral), level offsets r_n
        self.mv = M + 1 if layout == "vertex" else M
        self.r = {lev: 0 for lev in range(1, L + 1)} if layout == "vertex" else block_offsets(L, eta)

    # -- macropoints ---------------------------------------------------------
    def all_vertices(self):
        """all macropoints k ∈ {0..mv-1}^d (mv = M+1 vertex, M block), lexicographic, x fastest"""
        for rev in itertools.product(range(self.mv), repeat=self.d):
            yield tuple(reversed(rev))

    def num_macropoints(self) -> int:
        return self.mv ** self.d

    def linear_index(self, k) -> int:
        idx = 0
        for i in reversed(range(self.d)):
            idx = idx * self.mv + k[i]
        return idx

    def in_T(self, k, lev: int) -> bool:
        s = self.eta ** (self.L - lev)
        return all(ki % s == self.r[lev] for ki in k)

    def level_of(self, k) -> int:
        for lev in range(1, self.L + 1):
            if self.in_T(k, lev):
                return lev
        raise AssertionError

    def T(self, lev: int):
        return [k for k in self.all_vertices() if self.in_T(k, lev)]

    def S(self, lev: int):
        """Eq. (10): S_n = T_n minus the union of earlier S_k."""
        earlier = set()
        for m in range(1, lev):
            earlier.update(self.S(m))
        return [k for k in self.T(lev) if k not in earlier]

    # -- windows ---------------------------------------------------------------
    def origin2(self, ki: int) -> int:
        """2 × fine-cell coordinate of x_p along one dimension (vertex k·c, block k·c + c/2)"""
        return 2 * ki * self.c + (self.c if self.layout == "block" else 0)

    def l_of(self, k) -> int:
        """oversampling layers of macropoint k's window: l, except the level-1 points of the
        physical-coordinate variant (NEXT-4: "level-1 regions enlarged to the
        union of R_p^+ over all assigned children"): a child assigned to its nearest S_1 point lies
        within η^{L-1}H/2 of it per coordinate, so l + η^{L-1}/2 layers cover every child's window"""
        if self.interp == "physical_s1" and self.level_of(k) == 1:
            return self.l + self.eta ** (self.L - 1) // 2
        return self.l

    def window(self, k):
        """fine-cell box [lo, hi) per dimension of R_p^+ = x_p ± (l+½)H, clipped"""
        w2 = (2 * self.l_of(k) + 1) * self.c  # 2 × half width
        lo = tuple(max(0, (self.origin2(ki) - w2) // 2) for ki in k)
        hi = tuple(min(self.n, (self.origin2(ki) + w2) // 2) for ki in k)
        return lo, hi

    def subcell_coord(self, f: int) -> int:
        """index v of the subcell block containing fine cell f: dual block of vertex v
        [vc − c/2, vc + c/2) (vertex layout) or block v [vc, vc + c) (block layout)"""
        off = self.c // 2 if self.layout == "vertex" else 0
        return (f + off) // self.c

    def subcell_of_cell(self, k, cell):
        """local subcell index q of a global fine cell inside R_p^+"""
        q = 0
        lk = self.l_of(k)
        w = 2 * lk + 1
        for i in reversed(range(self.d)):
            v = self.subcell_coord(cell[i])
            slot = v - k[i] + lk
            assert 0 <= slot < w
            q = q * w + slot
        return q

    def centre_subcell(self, k=None) -> int:
        lk = self.l if k is None else self.l_of(k)
        w = 2 * lk + 1
        return sum(lk * w ** i for i in range(self.d))

    # -- hierarchy -------------------------------------------------------------
    def covers(self, t_i: int, k_i: int) -> bool:
        """1D: does the window of parent coordinate t_i cover child k_i's window in local
        coordinates (reading R9)?"""
        w2 = (2 * self.l + 1) * self.c

        def rng(v):
            o = self.origin2(v)
            return max(0, o - w2) - o, min(2 * self.n, o + w2) - o

        lo_p, hi_p = rng(k_i)
        lo_t, hi_t = rng(t_i)
        return lo_t <= lo_p and hi_t >= hi_p

    def _lattice_neighbours(self, ki: int, lev: int):
        """T_lev lattice coordinates bracketing ki: [(t, w)] (one point if ki is on the lattice or
        on one side only, weight 1; else two with linear weights)"""
        s, r = self.eta ** (self.L - lev), self.r[lev]
        if ki % s == r:
            return [(ki, 1.0)]
        a = ki - ((ki - r) % s)
        b = a + s
        pts = [t for t in (a, b) if 0 <= t < self.mv]
        if len(pts) == 1:
            return [(pts[0], 1.0)]
        wb = (ki - a) / s
        return [(a, 1.0 - wb), (b, wb)]

    def parents(self, k):
        """[(t, c_t)] for k ∈ S_n, n ≥ 2 (Eq. 11, reading R10 + R9 boundary rule).

        interp = "nearest_s1" (NEXT-1; "we only consider the first level for the
        interpolation operator, i.e. I_p = Φ_t with x_t ∈ S_1"): the single S_1 point nearest to
        x_p (Euclidean) among those whose window covers the child's (reading R9), weight 1; ties
        go to the smaller coordinate in each dimension."""
        lev = self.level_of(k)
        if lev == 1:
            return []
        if self.interp == "physical_s1":
            # NEXT-4: the nearest S_1 point (ties: the smaller coordinate), weight 1, evaluated at
            # physical coordinates; its enlarged window contains the child's (checked)
            t = []
            for ki in k:
                cands = [ti for ti, _ in self._lattice_neighbours(ki, 1)]
                t.append(min(cands, key=lambda ti: (abs(ti - ki), ti)))
            t = tuple(t)
            (plo, phi), (clo, chi) = self.window(t), self.window(k)
            if not all(plo[i] <= clo[i] and phi[i] >= chi[i] for i in range(self.d)):
                raise ValueError(f"parent {t} does not contain the window of {k}")
            return [(t, 1.0)]
        if self.interp == "nearest_s1":
            t = []
            for ki in k:
                cands = [ti for ti, _ in self._lattice_neighbours(ki, 1)]
                cands = [ti for ti in cands if self.covers(ti, ki)]
                if not cands:
                    raise ValueError(f"no covering parent for macropoint {k}")
                t.append(min(cands, key=lambda ti: (abs(ti - ki), ti)))
            return [(tuple(t), 1.0)]
        per_dim = []
        for ki in k:
            cands = self._lattice_neighbours(ki, lev - 1)
            keep = [(t, w) for (t, w) in cands if self.covers(t, ki)]
            if not keep:
                raise ValueError(f"no covering parent for macropoint {k}")
            if len(keep) < len(cands):
                keep = [(keep[0][0], 1.0)]
            per_dim.append(keep)
        out = []
        for combo in itertools.product(*reversed(per_dim)):
            combo = tuple(reversed(combo))
            t = tuple(ti for ti, _ in combo)
            w = 1.0
            for _, wi in combo:
                w *= wi
            out.append((t, w))
        return out


def block_centred_level_counts(blocks_per_dim: int, eta: int, L: int, d: int = 2):
    """NEXT-1 variant (paper Figs. 2-3): macropoints at block centres,
    T_n realised on the η^{L-n}H block grid.  Returns |S_1|..|S_L|."""
    counts = []
    prev = 0
    for lev in range(1, L + 1):
        per = blocks_per_dim // eta ** (L - lev)
        tn = per ** d
        counts.append(tn - prev)
        prev = tn
    return counts
