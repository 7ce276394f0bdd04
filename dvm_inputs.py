"""Seeded synthetic inputs for the five BASELINE.json configurations (c1-c5).

Shared by tests/, bench.py and smoke(); holds none of the method's arithmetic
(no collision operator, no direction table, no weights) -- only the input
recipes of DESIGN.md §3 (readings R12-R15): Gaussians/Maxwellians sampled on
the node-centred periodic grid v_j = (x_j - N/2) h, h = 2L/N, times a seeded
multiplicative perturbation.  numpy.random.default_rng(seed) (PCG64); draw
order is documented per config.  Layout [cells][N]...[N], last axis fastest.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    d: int
    N: int
    Nbar: int
    L: float
    cells: int
    kernel: int  # 0 = 2D Maxwell molecules, 1 = 3D hard spheres
    desc: str


CONFIGS = {
    "c1": Config("c1", 2, 16, 4, 8.0, 1, 0, "d=2 Maxwell, N=16, Nbar=4, two bumps at ±(1.5,0), 1% noise, seed 0"),
    "c2": Config("c2", 2, 64, 8, 8.0, 1, 0, "d=2 Maxwell, N=64, Nbar=8, bumps at ±(1.0,0), 1% noise, seed 0; +100 Euler steps"),
    "c3": Config("c3", 2, 256, 16, 8.0, 1, 0, "d=2 Maxwell, N=256, Nbar=16, 4-bump mixture in |v|<3, unit mass, seed 0"),
    "c4": Config("c4", 3, 32, 4, 8.0, 1, 1, "d=3 hard spheres, N=32, Nbar=4, bumps at ±(1.5,0,0), 1% noise, seed 0"),
    "c5": Config("c5", 3, 64, 8, 8.0, 512, 1, "d=3 hard spheres, N=64, Nbar=8, 512 cells of perturbed Maxwellians, seed 0"),
}


def velocities(d: int, N: int, L: float = 8.0) -> list[np.ndarray]:
    """Broadcastable per-axis node velocities v_j = (x_j - N/2) h (reading R3)."""
    h = 2.0 * L / N
    v = (np.arange(N, dtype=np.float64) - N / 2) * h
    out = []
    for j in range(d):
        shape = [1] * d
        shape[j] = N
        out.append(v.reshape(shape))
    return out


def gaussian(d: int, N: int, L: float, centre, var: float = 1.0) -> np.ndarray:
    """Isotropic Gaussian density (2π var)^{-d/2} exp(-|v-c|²/(2 var)) on the grid."""
    vs = velocities(d, N, L)
    r2 = sum((vs[j] - centre[j]) ** 2 for j in range(d))
    return np.exp(-r2 / (2.0 * var)) / (2.0 * math.pi * var) ** (d / 2.0)


def two_bumps(d: int, N: int, L: float, sep_half: float, noise: float, seed: int) -> np.ndarray:
    """0.5 (G(v - c) + G(v + c)), c = (sep_half, 0, ...), times (1 + noise U(-1,1)).

    Draw order: one U(-1,1) per node in storage order (reading R12/R13)."""
    rng = np.random.default_rng(seed)
    c = [sep_half] + [0.0] * (d - 1)
    mc = [-x for x in c]
    f = 0.5 * (gaussian(d, N, L, c) + gaussian(d, N, L, mc))
    u = rng.uniform(-1.0, 1.0, size=f.shape)
    return f * (1.0 + noise * u)


def mixture4(N: int, L: float, seed: int) -> np.ndarray:
    """c3 (reading R14): 4 isotropic bumps, centres uniform in the disc |v|<3 by
    rejection from U(-3,3)^2 (all 4 centres first), then variances U(0.5,1.5);
    equal weights; renormalised so that h^2 sum f = 1."""
    rng = np.random.default_rng(seed)
    centres = []
    while len(centres) < 4:
        c = rng.uniform(-3.0, 3.0, size=2)
        if c[0] ** 2 + c[1] ** 2 < 9.0:
            centres.append(c)
    variances = rng.uniform(0.5, 1.5, size=4)
    f = sum(0.25 * gaussian(2, N, L, centres[b], variances[b]) for b in range(4))
    h = 2.0 * L / N
    return f / (h * h * f.sum())


def maxwellian_cells(ncells: int, N: int, L: float, noise: float, seed: int,
                     first_cell: int = 0) -> np.ndarray:
    """c5: per cell rho~U(0.5,1.5), u~U(-0.5,0.5)^3, T~U(0.8,1.2),
    M(rho,u,T)(v) = rho (2πT)^{-3/2} exp(-|v-u|²/2T), times
    (1 + noise U(-1,1)) per node.  Draw order per cell: rho, u_x, u_y, u_z, T,
    then N^3 node draws in storage order (reading R12).  Cells are generated in
    order; first_cell > 0 skips earlier cells' draws so a rank's shard is the
    same as the corresponding slice of the full batch."""
    rng = np.random.default_rng(seed)
    vs = velocities(3, N, L)
    out = np.empty((ncells, N, N, N), dtype=np.float64)
    for c in range(first_cell + ncells):
        rho = rng.uniform(0.5, 1.5)
        u = rng.uniform(-0.5, 0.5, size=3)
        T = rng.uniform(0.8, 1.2)
        noise_u = rng.uniform(-1.0, 1.0, size=(N, N, N))
        if c < first_cell:
            continue
        r2 = (vs[0] - u[0]) ** 2 + (vs[1] - u[1]) ** 2 + (vs[2] - u[2]) ** 2
        m = rho * np.exp(-r2 / (2.0 * T)) / (2.0 * math.pi * T) ** 1.5
        out[c - first_cell] = m * (1.0 + noise * noise_u)
    return out


def make(name: str, cells: int | None = None, first_cell: int = 0) -> np.ndarray:
    """Input of config `name` as float64 [cells, N^d] (c5 honours cells/first_cell)."""
    cfg = CONFIGS[name]
    nodes = cfg.N ** cfg.d
    if name == "c1":
        f = two_bumps(2, 16, cfg.L, 1.5, 0.01, 0)
    elif name == "c2":
        f = two_bumps(2, 64, cfg.L, 1.0, 0.01, 0)
    elif name == "c3":
        f = mixture4(256, cfg.L, 0)
    elif name == "c4":
        f = two_bumps(3, 32, cfg.L, 1.5, 0.01, 0)
    elif name == "c5":
        n = cfg.cells if cells is None else cells
        f = maxwellian_cells(n, 64, cfg.L, 0.02, 0, first_cell=first_cell)
    else:
        raise KeyError(name)
    return np.ascontiguousarray(f.reshape(-1, nodes))


def random_field(d: int, N: int, seed: int, positive: bool = True) -> np.ndarray:
    """Fuzz input: i.i.d. U(0,1) (or U(-1,1)) per node, shape [N]*d."""
    rng = np.random.default_rng(seed)
    lo = 0.0 if positive else -1.0
    return rng.uniform(lo, 1.0, size=(N,) * d)


def even_weights(d: int, Ntilde: int, seed: int, lo: float = 0.5, hi: float = 1.5) -> np.ndarray:
    """Seeded box table over [-Ñ,Ñ]^d (shape [2Ñ+1]*d, index k + Ñ) with
    w(-k) = w(k): synthetic decoupled weights a(k) or b(l) (eq:decoup)."""
    r = np.random.default_rng(seed).uniform(lo, hi, size=(2 * Ntilde + 1,) * d)
    return 0.5 * (r + np.flip(r))
