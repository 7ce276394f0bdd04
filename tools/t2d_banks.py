"""Shared-memory bank conflicts of phase A's T2D_e lookups in k_fg2 for the c5
directions under candidate table layouts: per direction, the mean number of
distinct-address wavefronts of a 16-lane phase (8-byte words, 16 banks of 8 B).
Usage: python tools/t2d_banks.py (needs a GPU for the plan's (u, w))."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1201_3986_b200 import Plan  # noqa: E402

p = Plan(3, 64, 8)
layouts = {
    "pu*64+pw": lambda pu, pw: pu * 64 + pw,
    "pu*65+pw": lambda pu, pw: pu * 65 + pw,
    "pu*64+(pw^pu&15)": lambda pu, pw: pu * 64 + (pw ^ (pu & 15)),
    "pu*64+(pw^(pu*5&15))": lambda pu, pw: pu * 64 + (pw ^ ((pu * 5) & 15)),
    "pu*66+pw": lambda pu, pw: pu * 66 + pw,
    "pu*64+(pw^(pu>>2&15))": lambda pu, pw: pu * 64 + (pw ^ ((pu >> 2) & 15)),
}
zl = np.arange(16)
res = {k: [] for k in layouts}
rng = np.random.default_rng(0)
for i in range(p.A):
    u, w, _ = p.geometry(i)
    for trial in range(8):
        g, yl, a, b = rng.integers(0, 64), rng.integers(0, 16), rng.integers(0, 4), rng.integers(0, 4)
        pu = (u[0] * g + u[1] * (yl + 16 * b) + u[2] * (zl + 16 * a)) & 63
        pw = (w[0] * g + w[1] * (yl + 16 * b) + w[2] * (zl + 16 * a)) & 63
        for k, f in layouts.items():
            idx = f(pu, pw)
            banks = {}
            for x in set(idx.tolist()):
                banks.setdefault(x % 16, set()).add(x)
            res[k].append(max(len(v) for v in banks.values()))
for k, v in res.items():
    print(f"{k:24s} mean wavefronts per 16-lane phase {np.mean(v):.3f}  (max {max(v)})")
