"""Parity margin of the default paths against the oracle on every BASELINE config
(c1-c4 full or sampled grids, c5 in bench.py's 512-cell launch on sampled nodes
of 4 cells): max |Q_gpu - Q_oracle| / max |Q_oracle| per config (bar: 1e-11).
Test infrastructure (calls oracle/); python tools/parity_margin.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dvm_inputs  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

rng = np.random.default_rng(11)
for name in ("c1", "c2", "c3", "c4", "c5"):
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    p = Plan(cfg.d, cfg.N, cfg.Nbar)
    q = p.collide(torch.from_numpy(f).cuda()).cpu().numpy()
    nodes = cfg.N ** cfg.d
    cells = [0] if f.shape[0] == 1 else [0, 1, 137, f.shape[0] - 1]
    worst = 0.0
    for c in cells:
        pts = None if nodes <= 4096 else np.sort(rng.choice(nodes, size=64 if name == "c5" else 400, replace=False))
        qo, _, _ = oracle.collide(f[c], cfg.d, cfg.N, cfg.Nbar, p.Ntilde, cfg.L, points=pts)
        qg = q[c] if pts is None else q[c][pts]
        worst = max(worst, float(np.abs(qg - qo[0]).max() / np.abs(qo[0]).max()))
    print(f"{name}: max rel err {worst:.2e} over {len(cells)} cell(s) ({'all' if nodes <= 4096 else 'sampled'} nodes)", flush=True)
