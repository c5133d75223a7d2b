"""Host post-processing of the validation workload (NEXT-3) on [P][N]-sized arrays.

The fine solve and the fine block averages run in libmch.so (mch_fine_solve,
mch_fine_block_averages); what remains is arithmetic on a few thousand numbers:

* macro block averages (1/|K_p|) int_{K_p} U_i of the upscaled Q1 solution U_i (block layout):
  the mean of the block's 2^d corner values;
* the relative L2 error e_2^(i) of PAPER.md:534-538 and the Type 1/2/3 comparisons of
  PAPER.md:539-545 (Type 1: L = 1 vs fine, Type 2: hierarchical vs fine, Type 3: hierarchical vs
  L = 1).
"""
from __future__ import annotations

import numpy as np


def macro_block_averages(U, d, M):
    """U [N][(M+1)^d] nodal (x fastest) -> [M^d][N] block means."""
    U = np.asarray(U)
    N = U.shape[0]
    grid = U.reshape((N,) + (M + 1,) * d)  # [N][z][y][x]
    acc = np.zeros((N,) + (M,) * d)
    for a in range(2 ** d):
        sl = tuple(slice((a >> (d - 1 - ax)) & 1, ((a >> (d - 1 - ax)) & 1) + M) for ax in range(d))
        acc += grid[(slice(None),) + sl]
    return (acc / 2 ** d).reshape(N, -1).T.copy()


def relative_l2_error(Ubar, ubar):
    """e_2 per continuum; entries where the reference is undefined (NaN) are skipped."""
    Ubar, ubar = np.asarray(Ubar), np.asarray(ubar)
    ok = np.isfinite(ubar)
    d = np.where(ok, Ubar - ubar, 0.0)
    r = np.where(ok, ubar, 0.0)
    return np.sqrt((d * d).sum(axis=0) / (r * r).sum(axis=0))
