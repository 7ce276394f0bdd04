"""Path 4 (FFT gain) vs path 2 (frame-plane gain) on 3D N = 64: max relative
difference and per-evaluation time (CUDA events, min and median of REPS).
Usage: python tools/fg_check.py NBAR CELLS   (env PATHS="2 4", REPS=4)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

nbar = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 18
reps = int(os.environ.get("REPS", "4"))
f = torch.from_numpy(dvm_inputs.make("c5", cells=cells)).cuda()
p = Plan(3, 64, nbar)
out = {}
for path in [int(x) for x in os.environ.get("PATHS", "2 4").split()]:
    p.set_path(path)
    q = p.collide(f)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q = p.collide(f)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    out[path] = q.cpu().numpy()
    print(f"path {path}: min {ts[0]:.2f} ms, median {ts[len(ts) // 2]:.2f} ms for {cells} cells "
          f"-> {cells / ts[0] * 1e3:.1f} cells/s", flush=True)
if 2 in out and 4 in out:
    d = np.abs(out[4] - out[2]).max() / np.abs(out[2]).max()
    print(f"max |Q4 - Q2| / max|Q2| = {d:.3e}")
