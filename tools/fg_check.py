"""Path 4 (FFT gain) vs path 2 (frame-plane gain) on 3D N = 64: max relative
difference and per-evaluation time.  Usage: python tools/fg_check.py NBAR CELLS"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

nbar = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 18
f = torch.from_numpy(dvm_inputs.make("c5", cells=cells)).cuda()
p = Plan(3, 64, nbar)
out = {}
for path in [int(x) for x in os.environ.get("PATHS", "2 4").split()]:
    p.set_path(path)
    q = p.collide(f)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 2
    for _ in range(reps):
        q = p.collide(f)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out[path] = q.cpu().numpy()
    print(f"path {path}: {dt * 1e3:.1f} ms for {cells} cells -> {cells / dt:.1f} cells/s", flush=True)
if 2 in out and 4 in out:
    d = np.abs(out[4] - out[2]).max() / np.abs(out[2]).max()
    print(f"max |Q4 - Q2| / max|Q2| = {d:.3e}")
