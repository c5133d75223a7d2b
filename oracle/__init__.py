"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementation of the hot path of hierarchical
multicontinuum homogenization (arXiv 2503.01276, Algorithm 1),
written from the paper with the readings listed in DESIGN.md §3 (SURVEY.md §8(c)
R1-R19).  It assembles every local saddle-point system explicitly (sparse Q1
stiffness, constraint rows, explicit prolongation P_n and Galerkin products
P_nᵀA₁P_n) and solves it by sparse direct LU (SciPy SuperLU) with one step of
iterative refinement.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2503_01276_b200``) never imports it, and the two share no code: the only
common module is ``mch_inputs`` (seeded κ/ψ generation, no method arithmetic).

Pinning status per function (details in DESIGN.md §4 and tests/test_oracle_*.py):
  planner.*        pinned (closed-form counts, paper Figs. 2-3 block-centred counts,
                   Table 1 oversampling layers, brute-force enumeration)
  fem.*            pinned (textbook Q1 matrices, quadrature, constants/linears)
  kkt.solve_kkt    pinned (1D hand solve, dense brute force)
  hmh.Oracle       pinned (dense brute force on tiny grids at L=1 and L=2, constant-κ
                   closed form 1.44, layered-media 1D reduction, partition of unity,
                   periodic invariance, energy optimality, L=1 ≡ plain)
  The effective-coefficient VALUES of the BASELINE configs: parity unpinned by the
  paper (it prints none); pinned only through the properties above.
"""
from .planner import Plan
from .hmh import Oracle

__all__ = ["Plan", "Oracle"]
