"""Context run for the paper's Table 2 workload: 2D, 100
TVD-RK2 steps (200 operator evaluations) of dt = 0.01 for N = 16 / 32 / 64 / 128
with the paper's box half-widths 5.5 / 7 / 8 / 8 and N̄ up to Ñ = ⌊N/(3+√2)⌋.
Timing only (a Gaussian datum; cost does not depend on the data).  The paper's
hardware and precision are not stated: context, not a target.
python tools/table2_context.py"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_3986_b200 import Plan  # noqa: E402

PAPER = {(16, 3): 0.5, (32, 3): 3.19, (32, 7): 14.52, (64, 3): 16.2, (64, 7): 73.4, (64, 14): 283.0,
         (128, 3): 85.8, (128, 7): 378.0, (128, 14): 1382.0, (128, 28): 5531.0}  # seconds, Table 2
HALF = {16: 5.5, 32: 7.0, 64: 8.0, 128: 8.0}
for (N, nb), tp in PAPER.items():
    L = HALF[N]
    h = 2 * L / N
    v = (np.arange(N) - N // 2) * h
    g = np.exp(-(v[:, None] ** 2 + v[None, :] ** 2) / 2) / (2 * math.pi)
    f = torch.from_numpy(g.reshape(1, -1).copy()).cuda()
    p = Plan(2, N, nb, L=L)
    p.rk2(f.clone(), 0.01, 3, moments=False)  # warm-up (workspaces, graph)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p.rk2(f, 0.01, 100, moments=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"N": N, "Nbar": nb, "Ntilde": p.Ntilde, "L": L, "rk2_100_steps_s": dt,
                      "paper_s": tp, "ratio": tp / dt}), flush=True)
