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

Lexicographic order: x (k[0]) fastest.
"""
from __future__ import annotations

import itertools
import math


def oversampling_layers_paper(H: float) -> int:
    """l = ⌈−2 log H⌉ with the natural log (§4; Table 1 prints 5, 7, 8
    for H = 1/12, 1/24, 1/48)."""
    return int(math.ceil(-2.0 * math.log(H) - 1e-12))


class Plan:
    def __init__(self, d: int, n: int, M: int, L: int, eta: int, l: int = 1, interp: str = "dlinear"):
        if n % M:
            raise ValueError("M must divide n (H/h integer)")
        self.d, self.n, self.M, self.L, self.eta, self.l = d, n, M, L, eta, l
        if interp not in ("dlinear", "nearest_s1"):
            raise ValueError("interp must be 'dlinear' or 'nearest_s1'")
        self.interp = interp
        self.c = n // M  # fine cells per H
        if self.c % 2:
            raise ValueError("H/(2h) must be an integer")
        if (self.c // 2) % (eta ** (L - 1)):
            raise ValueError("H/(2 h eta^(L-1)) must be an integer")
        if M % (eta ** (L - 1)):
            raise ValueError("eta^(L-1) must divide M")

    # -- macropoints ---------------------------------------------------------
    def all_vertices(self):
        """all k ∈ {0..M}^d, lexicographic, x fastest"""
        for rev in itertools.product(range(self.M + 1), repeat=self.d):
            yield tuple(reversed(rev))

    def linear_index(self, k) -> int:
        idx = 0
        for i in reversed(range(self.d)):
            idx = idx * (self.M + 1) + k[i]
        return idx

    def level_of(self, k) -> int:
        for lev in range(1, self.L + 1):
            s = self.eta ** (self.L - lev)
            if all(ki % s == 0 for ki in k):
                return lev
        raise AssertionError

    def T(self, lev: int):
        s = self.eta ** (self.L - lev)
        return [k for k in self.all_vertices() if all(ki % s == 0 for ki in k)]

    def S(self, lev: int):
        """Eq. (10): S_n = T_n minus the union of earlier S_k."""
        earlier = set()
        for m in range(1, lev):
            earlier.update(self.S(m))
        return [k for k in self.T(lev) if k not in earlier]

    # -- windows ---------------------------------------------------------------
    def window(self, k):
        """fine-cell box [lo, hi) per dimension of R_p^+"""
        half = (2 * self.l + 1) * self.c // 2
        lo = tuple(max(0, ki * self.c - half) for ki in k)
        hi = tuple(min(self.n, ki * self.c + half) for ki in k)
        return lo, hi

    def subcell_of_cell(self, k, cell):
        """local subcell index q of a global fine cell inside R_p^+ (dual block of vertex v)"""
        q = 0
        w = 2 * self.l + 1
        for i in reversed(range(self.d)):
            v = (cell[i] + self.c // 2) // self.c
            slot = v - k[i] + self.l
            assert 0 <= slot < w
            q = q * w + slot
        return q

    def centre_subcell(self) -> int:
        w = 2 * self.l + 1
        return sum(self.l * w ** i for i in range(self.d))

    # -- hierarchy -------------------------------------------------------------
    def covers(self, t_i: int, k_i: int) -> bool:
        """1D: does the window of parent coordinate t_i cover child k_i's window in local
        coordinates (reading R9)?"""
        half = (2 * self.l + 1) * self.c // 2
        lo_p = max(0, k_i * self.c - half) - k_i * self.c
        hi_p = min(self.n, k_i * self.c + half) - k_i * self.c
        lo_t = max(0, t_i * self.c - half) - t_i * self.c
        hi_t = min(self.n, t_i * self.c + half) - t_i * self.c
        return lo_t <= lo_p and hi_t >= hi_p

    def parents(self, k):
        """[(t, c_t)] for k ∈ S_n, n ≥ 2 (Eq. 11, reading R10 + R9 boundary rule).

        interp = "nearest_s1" (NEXT-1; "we only consider the first level for the
        interpolation operator, i.e. I_p = Φ_t with x_t ∈ S_1"): the single S_1 point nearest to
        x_p (Euclidean) among those whose window covers the child's (reading R9), weight 1; ties
        go to the smaller coordinate in each dimension."""
        lev = self.level_of(k)
        if lev == 1:
            return []
        if self.interp == "nearest_s1":
            s1 = self.eta ** (self.L - 1)  # spacing of T_1 = S_1 in macro units
            t = []
            for ki in k:
                a = (ki // s1) * s1
                cands = [a] if ki == a else [a, a + s1]
                cands = [ti for ti in cands if self.covers(ti, ki)]
                if not cands:
                    raise ValueError(f"no covering parent for macropoint {k}")
                t.append(min(cands, key=lambda ti: (abs(ti - ki), ti)))
            return [(tuple(t), 1.0)]
        s = self.eta ** (self.L - lev + 1)  # spacing of T_{n-1} in macro units
        per_dim = []
        for ki in k:
            if ki % s == 0:
                cands = [(ki, 1.0)]
            else:
                a = (ki // s) * s
                b = a + s
                wb = (ki - a) / s
                cands = [(a, 1.0 - wb), (b, wb)]
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
