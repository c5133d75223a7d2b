"""Seeded media generators for the BASELINE.json configurations.

Conventions (SURVEY.md §8(c) reading R14):

* Domain [0,1]^d, ``n`` fine cells per dimension, h = 1/n.  Cell (i0,..,i_{d-1})
  has centre ((i+1/2)h).  Arrays are numpy C-order with x fastest, i.e. shape
  ``(n,)*d`` indexed ``[z, y, x]`` (3D) or ``[y, x]`` (2D).
* ``kappa``: float64 > 0 per fine cell.  ``ids``: uint8 continuum id per fine cell
  (ψ_j = [ids == j], §2).
* Microstructure: ε-cells of ``eps_cells`` fine cells; each holds a centred disk
  (sphere) of radius r(x)·ε, r(x) = 0.25 + 0.1·Π_i sin(2π x_i) evaluated at the
  ε-cell centre; a fine cell is inside iff the squared distance of its centre to
  the ε-cell centre is < (rε)^2 (strict).
* Config 3 adds one horizontal channel per ε-row, x_2 ∈ [kε, kε + ε/8) (one fine
  cell at h = 1/2048), and a log-normal matrix κ = exp(0.5·G) with G a seeded
  random-Fourier-feature Gaussian field (squared-exponential covariance, length
  0.25), drawn with numpy's counter-based Philox generator.

Nothing in this module evaluates the homogenization method.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    d: int            # spatial dimension
    n: int            # fine cells per dimension (h = 1/n)
    M: int            # macro cells per dimension (H = 1/M); macropoints = (M+1)^d vertices
    L: int            # hierarchy levels
    eta: int          # coarsening factor
    N: int            # number of continua
    eps_cells: int    # fine cells per ε-cell of the microstructure
    matrix: str       # "sin1" | "sincos" | "one" | "lognormal"
    k_incl: float     # κ in inclusions (continuum 1)
    k_channel: float = 0.0  # κ in channels (continuum 2), config 3 only
    seed: int = 0
    l: int = 1        # oversampling layers (R_p^+ = x_p ± (l+1/2)H), SURVEY R2

    @property
    def n_rhs(self) -> int:
        return self.N * (1 + self.d)

    @property
    def c(self) -> int:
        """fine cells per macro cell H"""
        return self.n // self.M


# BASELINE.json "configs" (index 1..5); SURVEY.md §8(d) table.
CONFIGS = {
    1: Config("c1", 2, 256, 8, 1, 2, 2, 8, "sin1", 100.0, seed=0),
    2: Config("c2", 2, 1024, 32, 3, 2, 2, 8, "sin1", 1e3, seed=1),
    3: Config("c3", 2, 2048, 64, 3, 2, 3, 8, "lognormal", 100.0, k_channel=1e4, seed=2),
    4: Config("c4", 3, 128, 8, 2, 2, 2, 8, "one", 100.0, seed=3),
    5: Config("c5", 3, 256, 16, 4, 2, 2, 8, "sincos", 1e3, seed=4),
}


def _centres(n: int) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 0.5) / n


def _grid(d: int, n: int):
    """Cell-centre coordinate arrays x_0..x_{d-1}, each broadcastable to shape (n,)*d [.., x]."""
    c = _centres(n)
    out = []
    for i in range(d):
        shape = [1] * d
        shape[d - 1 - i] = n
        out.append(c.reshape(shape))
    return out


def _lognormal_field(d: int, n: int, seed: int, length: float = 0.25, sigma: float = 0.5,
                     features: int = 256) -> np.ndarray:
    """κ = exp(σ G), G ≈ unit-variance SE-covariance field via random Fourier features."""
    rng = np.random.Generator(np.random.Philox(seed))
    omega = rng.standard_normal((features, d)) / length
    phase = rng.uniform(0.0, 2.0 * math.pi, features)
    c = _centres(n)
    if d == 2:
        a = np.exp(1j * np.outer(c, omega[:, 1]))                       # (ny, F)
        b = np.exp(1j * (np.outer(omega[:, 0], c) + phase[:, None]))    # (F, nx)
        g = np.real(a @ b)
    else:
        g = np.zeros((n, n, n))
        bx = np.exp(1j * (np.outer(omega[:, 0], c) + phase[:, None]))  # (F, nx)
        for iz in range(n):
            a = np.exp(1j * (np.outer(c, omega[:, 1]) + c[iz] * omega[:, 2]))
            g[iz] = np.real(a @ bx)
    g *= math.sqrt(2.0 / features)
    return np.exp(sigma * g)


def make_medium(cfg: Config):
    """Return (kappa float64, ids uint8), both shape (n,)*d, x fastest."""
    d, n, e = cfg.d, cfg.n, cfg.eps_cells
    if n % e:
        raise ValueError("eps_cells must divide n")
    xs = _grid(d, n)
    shape = (n,) * d
    # matrix κ at fine-cell centres
    if cfg.matrix == "one":
        km = np.ones(shape)
    elif cfg.matrix == "sin1":
        km = np.broadcast_to(1.0 + 0.5 * np.sin(np.pi * xs[0]), shape).copy()
    elif cfg.matrix == "sincos":
        km = np.broadcast_to(1.0 + 0.5 * np.sin(np.pi * xs[0]) * np.cos(np.pi * xs[1]), shape).copy()
    elif cfg.matrix == "lognormal":
        km = _lognormal_field(d, n, cfg.seed)
    else:
        raise ValueError(cfg.matrix)
    # inclusion radius r at ε-cell centres, offsets of fine centres within the ε-cell (ε units)
    neps = n // e
    ce = (np.arange(neps, dtype=np.float64) + 0.5) / neps
    off = (np.arange(e, dtype=np.float64) + 0.5) / e - 0.5
    # per-axis: epsilon-cell index and offset of every fine cell
    idx = np.arange(n)
    eidx, oidx = idx // e, idx % e
    prod = np.ones(shape)
    dist2 = np.zeros(shape)
    for i in range(d):
        sh = [1] * d
        sh[d - 1 - i] = n
        prod = prod * np.sin(2.0 * np.pi * ce[eidx]).reshape(sh)
        dist2 = dist2 + (off[oidx] ** 2).reshape(sh)
    r = 0.25 + 0.1 * prod
    incl = dist2 < r * r
    ids = np.zeros(shape, dtype=np.uint8)
    kappa = km.copy()
    ids[incl] = 1
    kappa[incl] = cfg.k_incl
    if cfg.k_channel:
        if d != 2:
            raise ValueError("channels are a 2D config-3 feature")
        rows = (np.arange(n) % e) < max(1, e // 8)
        ids[rows, :] = 2
        kappa[rows, :] = cfg.k_channel
    return np.ascontiguousarray(kappa), np.ascontiguousarray(ids)


def random_medium(d: int, n: int, N: int, seed: int, kmin: float = 1.0, kmax: float = 100.0,
                  block: int = 1):
    """Random cellwise κ ∈ [kmin,kmax] (log-uniform) and random ids in [0,N) (constant on
    ``block``^d cell groups).  Used by the tiny brute-force tests."""
    rng = np.random.Generator(np.random.Philox(seed))
    shape = (n,) * d
    kappa = np.exp(rng.uniform(math.log(kmin), math.log(kmax), shape))
    nb = n // block
    ids_c = rng.integers(0, N, (nb,) * d).astype(np.uint8)
    ids = ids_c
    for ax in range(d):
        ids = np.repeat(ids, block, axis=ax)
    return np.ascontiguousarray(kappa), np.ascontiguousarray(ids)


def layered_medium(d: int, n: int, period: int, kappas, widths):
    """Layers normal to x_{d-1} (the last coordinate): within each period of ``period``
    fine cells, continuum j occupies ``widths[j]`` consecutive cell rows with κ = kappas[j]."""
    assert sum(widths) == period
    shape = (n,) * d
    lay = np.zeros(period, dtype=np.uint8)
    pos = 0
    for j, w in enumerate(widths):
        lay[pos:pos + w] = j
        pos += w
    row_id = lay[np.arange(n) % period]
    sh = [1] * d
    sh[0] = n  # first numpy axis = last coordinate
    ids = np.broadcast_to(row_id.reshape(sh), shape).astype(np.uint8).copy()
    kappa = np.asarray(kappas, dtype=np.float64)[ids]
    return np.ascontiguousarray(kappa), np.ascontiguousarray(ids)


def periodic_medium(d: int, n: int, period: int, radius: float, k_matrix: float, k_incl: float):
    """Centred disk/sphere of radius ``radius`` (period units) in every period cell, constant κ."""
    off = (np.arange(period, dtype=np.float64) + 0.5) / period - 0.5
    idx = np.arange(n) % period
    shape = (n,) * d
    dist2 = np.zeros(shape)
    for i in range(d):
        sh = [1] * d
        sh[d - 1 - i] = n
        dist2 = dist2 + (off[idx] ** 2).reshape(sh)
    incl = dist2 < radius * radius
    ids = incl.astype(np.uint8)
    kappa = np.where(incl, k_incl, k_matrix).astype(np.float64)
    return np.ascontiguousarray(kappa), np.ascontiguousarray(ids)


def paper_source(d: int, n: int, ids, eps: float, low=(0,)):
    """Source of the paper's experiments at fine-cell centres:
    f = e^{-40((x_1-1/2)^2 + (x_2-1/2)^2)}, scaled by ε/10 in the low-conductivity region Ω_1
    (cells whose continuum id is in ``low``; continuum 0, the matrix, in the BASELINE media).
    The paper's f depends on x_1, x_2 only; in 3D the same formula is used (reading R24)."""
    xs = _grid(d, n)
    shape = (n,) * d
    g = np.broadcast_to(np.exp(-40.0 * ((xs[0] - 0.5) ** 2 + (xs[1] - 0.5) ** 2)), shape).copy()
    ids = np.asarray(ids).reshape(shape)
    in_low = np.isin(ids, np.asarray(low, dtype=ids.dtype))
    g[in_low] *= eps / 10.0
    return np.ascontiguousarray(g)


def paper_medium(d: int, n: int, eps: float, geometry: str = "layered"):
    """The paper's permeability κ = g1·g2 at fine-cell centres:
    g1 = 2 + sin(πx_1) sin(πx_2); g2 = ε/10⁴ in the low-conductivity region Ω_1 (continuum 0),
    1/(100ε) in Ω_2 (continuum 1).  The geometries are figures in the paper (reading R25):
    "layered" = layers normal to x_2 of period ε, Ω_2 the upper half of each period;
    "crossed" = Ω_2 the union of the x_2-layers and the same layers normal to x_1."""
    xs = _grid(d, n)
    shape = (n,) * d
    g1 = np.broadcast_to(2.0 + np.sin(np.pi * xs[0]) * np.sin(np.pi * xs[1]), shape)
    ph = [np.broadcast_to((xs[i] / eps) % 1.0 >= 0.5, shape) for i in range(2)]
    hi = ph[1] if geometry == "layered" else (ph[0] | ph[1])
    ids = hi.astype(np.uint8)
    kappa = g1 * np.where(hi, 1.0 / (100.0 * eps), eps / 1e4)
    return np.ascontiguousarray(kappa), np.ascontiguousarray(ids)
