"""Per-direction cross-check of the cluster path against the orbit path (GPU debug)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1201_3986_b200 import Plan

for N, Nb, Nt, cells in [(32, 1, 4, 1), (64, 1, 4, 1), (64, 1, 4, 20)]:
    full = Plan(3, N, Nb, Ntilde=Nt)
    A = full.A
    f = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, size=(cells, N ** 3))).cuda()
    dirs = full.directions()[0]
    print(f"N={N} Nb={Nb} Nt={Nt} cells={cells} A={A}", flush=True)
    for r in range(A):
        p = Plan(3, N, Nb, Ntilde=Nt, shard_rank=r, shard_world=A)
        loc = np.nonzero(p.directions()[3])[0]
        q2 = p.collide(f).cpu().numpy()
        p.set_path(1)
        q1 = p.collide(f).cpu().numpy()
        err = np.abs(q2 - q1).max() / max(np.abs(q1).max(), 1e-300)
        i = int(loc[0])
        u, w, rows = p.geometry(i)
        print(f"  dir {i} e={dirs[i]} u={u} w={w} rows={len(rows)} rel={err:.2e}", flush=True)
