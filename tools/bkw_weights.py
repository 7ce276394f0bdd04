"""Which decoupled weight a(k) b(l) makes libdvm's operator the 2D Maxwell
molecules operator of the BKW solution?  For a(k) on the box [-Ñ,Ñ]^2 this
prints, per grid, the least-squares constant c of c Q(f_BKW(0)) ≈ d/dt f_BKW(0)
and the relative L1 residual of that fit (0 for a consistent kernel, up to
discretisation error).  Candidates: the built-in h^3 |k| / gcd(k) (PAPER.md:
582-587) and the lattice discretisation of the Carleman integral with a
constant B̃ = 2B = 1/π, a(k) = h^2 / (π gcd(k)) (reading R24).
Usage: python tools/bkw_weights.py"""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3986_b200 import Plan, bkw  # noqa: E402


def box_weights(Nt, h, kind):
    a = np.zeros((2 * Nt + 1, 2 * Nt + 1))
    for i in range(-Nt, Nt + 1):
        for j in range(-Nt, Nt + 1):
            if i == 0 and j == 0:
                continue
            g = math.gcd(abs(i), abs(j))
            a[i + Nt, j + Nt] = h ** 3 * math.hypot(i, j) / g if kind == "paper" else h ** 2 / (math.pi * g)
    return a


for N in (16, 32, 64, 128):
    T = bkw.PAPER_BOX[N]
    probe = Plan(2, N, 1, L=T)
    Nt = probe.Ntilde
    h = 2 * T / N
    v2 = bkw.grid_v2(N, T)
    f0 = torch.from_numpy(bkw.f_exact(0.0, v2).reshape(-1)).cuda()
    ft = bkw.dfdt_exact(0.0, v2).reshape(-1)
    for kind in ("paper", "carleman"):
        p = Plan(2, N, Nt, L=T)
        p.set_weights(box_weights(Nt, h, kind), None)
        q = p.collide(f0).cpu().numpy()
        c = float(np.dot(q, ft) / np.dot(q, q))
        res = np.abs(c * q - ft).sum() / np.abs(ft).sum()
        res1 = np.abs(q - ft).sum() / np.abs(ft).sum()
        print(f"N={N:4d} T={T} Ñ={Nt:3d} {kind:9s}: c = {c:.6f}, L1 residual of the fit {res:.3e}, "
              f"residual at c = 1: {res1:.3e}", flush=True)
