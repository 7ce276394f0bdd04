"""Space-inhomogeneous use of the operator with a space-dependent N̄
(PAPER.md:904-911): a 1D periodic space grid of X cells, a 2D velocity grid per
cell, Strang-free first-order splitting  f <- T(dt) f,  f <- f + dt Q_{N̄(x)}(f)
with T the upwind transport of  ∂_t f + v_x ∂_x f = 0  (torch on the device,
plumbing: not the operator) and Q evaluated per cell by
dvm_collide_batched_levels with N̄ chosen each step by the reference policy
(`equilibrium_levels`: cells close to their local Maxwellian get the low level).

Reports per step: the share of cells at each level, the time of the collision
call against the uniform-max-N̄ call on the same f, mass drift, and at the end
the L1 difference between the adaptive and the uniform-N̄ trajectories.

Usage: python tools/inhomogeneous.py [X] [steps] [N] [low N̄] [high N̄]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1201_3986_b200 import Plan  # noqa: E402
from paper_1201_3986_b200.adaptive import AdaptiveNbar, equilibrium_levels  # noqa: E402

X = int(sys.argv[1]) if len(sys.argv) > 1 else 128
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
N = int(sys.argv[3]) if len(sys.argv) > 3 else 32
levels = [int(sys.argv[4]) if len(sys.argv) > 4 else 2, int(sys.argv[5]) if len(sys.argv) > 5 else 7]
L, thresholds = 8.0, [0.02]
h = 2 * L / N
dx = 1.0 / X
v = (torch.arange(N, dtype=torch.float64) - N // 2) * h
VX, VY = torch.meshgrid(v, v, indexing="ij")
vmax = float(v.abs().max())
dt = 0.5 * dx / vmax  # CFL 1/2 for the upwind transport


def maxwellian(rho, ux, T):
    return rho / (2 * np.pi * T) * torch.exp(-((VX - ux) ** 2 + VY ** 2) / (2 * T))


# near-equilibrium density wave everywhere, a two-stream non-equilibrium slab in the middle
xs = (np.arange(X) + 0.5) * dx
cells = []
for x in xs:
    f = maxwellian(1.0 + 0.3 * np.sin(2 * np.pi * x), 0.0, 1.0)
    if 0.4 < x < 0.6:
        f = 0.5 * (maxwellian(1.0, 1.2, 0.5) + maxwellian(1.0, -1.2, 0.5))
    cells.append(f.reshape(-1))
f0 = torch.stack(cells).cuda()
VXd = VX.reshape(-1).cuda()


def transport(f):
    """First-order upwind in x (periodic), per velocity node."""
    pos = (VXd > 0).to(f.dtype)
    back = f - torch.roll(f, 1, 0)    # f_i − f_{i−1}
    fwd = torch.roll(f, -1, 0) - f    # f_{i+1} − f_i
    return f - dt / dx * VXd * (pos * back + (1 - pos) * fwd)


ad = AdaptiveNbar(2, N, levels)
full = Plan(2, N, levels[-1], Ntilde=ad.Ntilde)
print(f"X = {X} cells of {N}^2 velocities, levels {levels} (A = {ad.directions()}), Ñ = {ad.Ntilde}, "
      f"dt = {dt:.3e}, {steps} steps")
fa, fu = f0.clone(), f0.clone()
mass0 = float(fa.sum()) * h * h * dx
t_ad = t_full = 0.0
for s in range(steps):
    fa, fu = transport(fa), transport(fu)
    nb, delta = equilibrium_levels(fa, 2, N, L, levels, thresholds)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qa = ad.collide(fa, nb)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    qu = full.collide(fu)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    t_ad += t1 - t0
    t_full += t2 - t1
    fa += dt * qa
    fu += dt * qu
    if s % 10 == 0 or s == steps - 1:
        share = {lv: float(np.mean(nb == lv)) for lv in levels}
        drift = abs(float(fa.sum()) * h * h * dx - mass0) / mass0
        print(f"step {s:3d}: level share {share}, mass drift {drift:.1e}, "
              f"collision {1e3 * (t1 - t0):.2f} ms adaptive / {1e3 * (t2 - t1):.2f} ms uniform", flush=True)
diff = float((fa - fu).abs().sum() / fu.abs().sum())
print(f"after {steps} steps: relative L1 difference adaptive vs uniform N̄ = {diff:.2e}; "
      f"collision time {1e3 * t_ad:.1f} ms adaptive vs {1e3 * t_full:.1f} ms uniform")
