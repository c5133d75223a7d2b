"""Pins for oracle/planner.py (macrogrid hierarchy, §3.1)."""
import itertools
import json
import math
import os

import pytest

from mch_inputs import CONFIGS
from oracle.planner import Plan, block_centred_level_counts, oversampling_layers_paper

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_paper_fig2_3_block_centred_counts():
    g = json.load(open(os.path.join(GOLDEN, "paper_fig2_3_level_counts.json")))
    assert block_centred_level_counts(g["blocks_per_dim"], g["eta"], g["L"]) == g["S_counts"]


def test_paper_table1_oversampling_layers():
    g = json.load(open(os.path.join(GOLDEN, "paper_table1_oversampling.json")))
    assert [oversampling_layers_paper(1.0 / Hi) for Hi in g["H_inverse"]] == g["l"]


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_level_counts_closed_form(cid):
    """|T_n| = (M/η^{L-n} + 1)^d (vertex grid of spacing η^{L-n}H) and |S_n| = |T_n| − |T_{n-1}|
    (Eq. 10 with S_{n+1} = T_{n+1} \\ T_n)."""
    cfg = CONFIGS[cid]
    p = Plan(cfg.d, cfg.n, cfg.M, cfg.L, cfg.eta, cfg.l)
    prev = 0
    total = 0
    for lev in range(1, cfg.L + 1):
        tn = (cfg.M // cfg.eta ** (cfg.L - lev) + 1) ** cfg.d
        S = p.S(lev)
        assert len(S) == tn - prev
        assert len(set(S)) == len(S)
        prev = tn
        total += len(S)
    assert total == (cfg.M + 1) ** cfg.d


def test_level_counts_survey_table():
    # SURVEY.md §8(a) table (same closed form, spelled out)
    want = {1: [81], 2: [81, 208, 800], 3: [289, 800, 3136], 4: [125, 604], 5: [27, 98, 604, 4184]}
    for cid, counts in want.items():
        cfg = CONFIGS[cid]
        p = Plan(cfg.d, cfg.n, cfg.M, cfg.L, cfg.eta, cfg.l)
        assert [len(p.S(l)) for l in range(1, cfg.L + 1)] == counts


@pytest.mark.parametrize("d,M,L,eta", [(2, 32, 3, 2), (2, 8, 2, 2), (3, 16, 4, 2), (2, 9, 2, 3)])
def test_parents_brute_force(d, M, L, eta):
    """Parents: subset of T_{n-1} inside the T_{n-1} cell containing x_p, weights sum to 1,
    dense property dist < η^{L-n+1}H·√d, and every parent window covers the
    child's window after the local-coordinate shift (reading R9), checked by brute force."""
    c = 2 * eta ** (L - 1) * 2
    n = M * c
    p = Plan(d, n, M, L, eta)
    for lev in range(2, L + 1):
        Tprev = set(p.T(lev - 1))
        s = eta ** (L - lev + 1)
        for k in p.S(lev):
            par = p.parents(k)
            assert abs(sum(w for _, w in par) - 1.0) < 1e-14
            lo_k, hi_k = p.window(k)
            for t, w in par:
                assert t in Tprev and w > 0
                assert max(abs(a - b) for a, b in zip(t, k)) <= s
                assert math.dist(t, k) < s * math.sqrt(d) + 1e-12
                lo_t, hi_t = p.window(t)
                for i in range(d):
                    assert lo_t[i] - t[i] * c <= lo_k[i] - k[i] * c
                    assert hi_t[i] - t[i] * c >= hi_k[i] - k[i] * c


def test_parent_weights_interior_eta2():
    """η = 2 interior children: weights ½ per off-lattice coordinate (d-linear interpolation)."""
    p = Plan(2, 1024, 32, 3, 2)
    par = dict(p.parents((6, 4)))     # level 2 child: x off the T_1 lattice (spacing 4)
    assert par == {(4, 4): 0.5, (8, 4): 0.5}
    par = dict(p.parents((5, 5)))     # level 3 child, both coordinates off the T_2 lattice
    assert par == {(4, 4): 0.25, (6, 4): 0.25, (4, 6): 0.25, (6, 6): 0.25}
    # boundary rule: parent on ∂Ω dropped, weight to the opposite parent
    par = dict(p.parents((2, 4)))
    assert par == {(4, 4): 1.0}


def test_divisibility_errors():
    with pytest.raises(ValueError):
        Plan(2, 100, 8, 1, 2)       # M ∤ n
    with pytest.raises(ValueError):
        Plan(2, 64, 16, 3, 2)       # H/(2hη^{L-1}) not integer (c = 4)
    with pytest.raises(ValueError):
        Plan(2, 96, 12, 4, 2)       # η^{L-1} = 8 ∤ M


def test_subcell_partition():
    """Subcells R_q tile R_p^+ (every window cell has exactly one subcell; K_p is the centre)."""
    p = Plan(2, 64, 8, 1, 2)
    for k in [(0, 0), (3, 4), (8, 8)]:
        lo, hi = p.window(k)
        for cell in itertools.product(range(lo[0], hi[0]), range(lo[1], hi[1])):
            q = p.subcell_of_cell(k, cell)
            v = tuple(k[i] + (q // 3 ** i) % 3 - 1 for i in range(2))
            assert all(abs(cell[i] + 0.5 - v[i] * p.c) <= p.c / 2 for i in range(2))


@pytest.mark.parametrize("d,n,M,L,eta", [(2, 64, 8, 3, 2), (2, 72, 12, 2, 3), (3, 64, 8, 3, 2)])
def test_nearest_s1_parents_brute_force(d, n, M, L, eta):
    """NEXT-1, PAPER.md:425 (I_p = Φ_t, x_t ∈ S_1): brute force over every S_1 point — the chosen
    parent is in S_1, its window covers the child's in local coordinates (reading R9), it is the
    nearest such point (Euclidean), ties resolved to the smallest coordinates; weight 1."""
    p = Plan(d, n, M, L, eta, interp="nearest_s1")
    s1 = set(p.S(1))
    for k in p.all_vertices():
        par = p.parents(k)
        if p.level_of(k) == 1:
            assert par == []
            continue
        assert len(par) == 1 and par[0][1] == 1.0
        t = par[0][0]
        assert t in s1
        ok = [u for u in s1 if all(p.covers(u[i], k[i]) for i in range(d))]
        dist = lambda u: sum((u[i] - k[i]) ** 2 for i in range(d))
        best = min(dist(u) for u in ok)
        assert dist(t) == best
        ties = [u for u in ok if dist(u) == best]
        assert all(t[i] == min(u[i] for u in ties) for i in range(d)), (k, t, ties)


def test_paper_fig2_block_centred_positions():
    """Block-centred layout (NEXT-1): T_n reproduces the star positions of the paper's Figure 2
    (golden fixture with the tikz coordinates) and the S_n counts 4/12/48 of Figure 3."""
    g = json.load(open(os.path.join(GOLDEN, "paper_fig2_block_T_positions.json")))
    p = Plan(2, 8 * g["M"], g["M"], g["L"], g["eta"], layout="block")
    for lev in range(1, g["L"] + 1):
        idx = g["T_block_indices_per_dim"][str(lev)]
        assert sorted(p.T(lev)) == sorted(itertools.product(idx, repeat=2))
    c = json.load(open(os.path.join(GOLDEN, "paper_fig2_3_level_counts.json")))
    assert [len(p.S(lev)) for lev in range(1, 4)] == c["S_counts"]


@pytest.mark.parametrize("d,M,L,eta", [(2, 8, 3, 2), (2, 9, 3, 3), (2, 16, 4, 2), (3, 8, 3, 2)])
def test_block_levels_and_parents_brute_force(d, M, L, eta):
    """block layout: T_n from the oracle's modular rule equals the brute-force enumeration of coarse
    blocks (tests/bruteforce.py), and the oracle's parents equal the brute force's."""
    from tests.bruteforce import BruteForce
    import numpy as np
    n = M * eta ** (L - 1) * 2
    p = Plan(d, n, M, L, eta, layout="block")
    bf = BruteForce(d, n, M, L, eta, 1, np.ones((n,) * d), np.zeros((n,) * d, dtype=np.uint8),
                    layout="block")
    for lev in range(1, L + 1):
        assert set(p.T(lev)) == bf.Tsets[lev]
    for k in p.all_vertices():
        if p.level_of(k) == 1:
            continue
        a = sorted((t, round(w, 12)) for t, w in p.parents(k))
        b = sorted((t, round(w, 12)) for t, w in bf.parents(k))
        assert a == b, (k, a, b)
