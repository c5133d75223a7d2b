"""Oracle Q1 finite-element pieces (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

* Q1 element stiffness of the cube of side h: ∫_e ∇N_a·∇N_b written as the exact
  tensor sum Σ_k (1D stiffness in x_k) ⊗ (1D mass in the other coordinates)
  (weak form Eq. 2; cellwise κ).
* A₁ = Σ_e κ_e K_e on a box of fine cells, natural boundary conditions (reading R3).
* Constraint rows ℓ_qj(v) = ∫_{R_q} ψ_j v = Σ_{e⊂R_q, id_e=j} (h^d/2^d) Σ_corners v
  (Eq. 3/4 constraint lines; exact for Q1 and cellwise ψ).
* P_n: tensor product of 1D linear interpolation from the mesh hη^{n-1} to h
  (nested spaces V_n ⊂ V_1).

Node numbering inside a box with cell shape (n_0, .., n_{d-1}) (x first): node
(i_0, .., i_{d-1}) ↦ i_0 + (n_0+1)(i_1 + (n_1+1) i_2).  Element corner a has bits
a_i (x = bit 0).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def q1_stiffness_1d(h: float) -> np.ndarray:
    return np.array([[1.0, -1.0], [-1.0, 1.0]]) / h


def q1_mass_1d(h: float) -> np.ndarray:
    return np.array([[2.0, 1.0], [1.0, 2.0]]) * (h / 6.0)


def q1_element_stiffness(d: int, h: float) -> np.ndarray:
    """2^d × 2^d, corner index a = Σ a_i 2^i (x fastest)."""
    K = np.zeros((2 ** d, 2 ** d))
    for k in range(d):
        mats = [q1_stiffness_1d(h) if i == k else q1_mass_1d(h) for i in range(d)]
        T = np.ones((1, 1))
        for i in range(d):  # kron(A_last, ..., A_0) -> index = Σ a_i 2^i
            T = np.kron(mats[i], T)
        K += T
    return K


def _node_ids(cells_shape_x_first):
    """(n_elem, 2^d) array of corner node ids, elements enumerated x fastest."""
    d = len(cells_shape_x_first)
    nn = [s + 1 for s in cells_shape_x_first]
    strides = [1]
    for i in range(1, d):
        strides.append(strides[-1] * nn[i - 1])
    grids = np.meshgrid(*[np.arange(s) for s in reversed(cells_shape_x_first)], indexing="ij")
    base = np.zeros(grids[0].shape, dtype=np.int64)
    for i in range(d):
        base += grids[d - 1 - i] * strides[i]
    base = base.reshape(-1)
    corners = []
    for a in range(2 ** d):
        off = sum(((a >> i) & 1) * strides[i] for i in range(d))
        corners.append(base + off)
    return np.stack(corners, axis=1), int(np.prod(nn))


def assemble_stiffness(kappa_box: np.ndarray, h: float, mask: np.ndarray | None = None) -> sp.csr_matrix:
    """A = Σ_e κ_e K_e over the cells of ``kappa_box`` (numpy shape [.., y, x]); only cells
    with mask True if given (used for the K_p-restricted Gram, Eq. 7)."""
    d = kappa_box.ndim
    shape_x_first = tuple(reversed(kappa_box.shape))
    nodes, nn = _node_ids(shape_x_first)
    Ke = q1_element_stiffness(d, h)
    kap = kappa_box.reshape(-1)
    if mask is not None:
        sel = mask.reshape(-1)
        nodes, kap = nodes[sel], kap[sel]
    rows = np.repeat(nodes, 2 ** d, axis=1).reshape(-1)
    cols = np.tile(nodes, (1, 2 ** d)).reshape(-1)
    vals = (kap[:, None] * Ke.reshape(1, -1)).reshape(-1)
    return sp.coo_matrix((vals, (rows, cols)), shape=(nn, nn)).tocsr()


def assemble_constraints(ids_box: np.ndarray, sub_box: np.ndarray, n_sub: int, N: int, h: float):
    """C₁ with rows r = q*N + j; returns (C csr [n_sub*N, nodes], measures V[r] = ∫_{R_q} ψ_j)."""
    d = ids_box.ndim
    shape_x_first = tuple(reversed(ids_box.shape))
    nodes, nn = _node_ids(shape_x_first)
    row_e = (sub_box.reshape(-1).astype(np.int64) * N + ids_box.reshape(-1).astype(np.int64))
    w = h ** d / 2 ** d
    rows = np.repeat(row_e, 2 ** d)
    cols = nodes.reshape(-1)
    vals = np.full(rows.shape, w)
    C = sp.coo_matrix((vals, (rows, cols)), shape=(n_sub * N, nn)).tocsr()
    V = np.bincount(row_e, minlength=n_sub * N).astype(np.float64) * h ** d
    return C, V


def prolongation_1d(n_coarse_cells: int, s: int) -> sp.csr_matrix:
    """(n_coarse_cells*s + 1) × (n_coarse_cells + 1) linear interpolation, coarse spacing s·h."""
    nf = n_coarse_cells * s + 1
    rows, cols, vals = [], [], []
    for i in range(nf):
        ic, rem = divmod(i, s)
        t = rem / s
        rows.append(i); cols.append(ic); vals.append(1.0 - t)
        if rem:
            rows.append(i); cols.append(ic + 1); vals.append(t)
    return sp.coo_matrix((vals, (rows, cols)), shape=(nf, n_coarse_cells + 1)).tocsr()


def prolongation(cells_shape_x_first, s: int) -> sp.csr_matrix:
    """tensor-product P_n for a box whose fine cell counts are divisible by s."""
    P = sp.identity(1, format="csr")
    for nc in cells_shape_x_first:
        if nc % s:
            raise ValueError("window not aligned with the level mesh")
        P = sp.kron(prolongation_1d(nc // s, s), P, format="csr")
    return P
