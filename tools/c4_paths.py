"""c4 (3D N = 32, N̄ = 4, one cell): per-evaluation time of the frame-plane
kernel (path 2) and the direction-pair spectral gain (path 6), CUDA events,
min of 20, plus their agreement.  Usage: python tools/c4_paths.py [CELLS]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1
f = torch.from_numpy(np.concatenate([dvm_inputs.make("c4")] * cells)).cuda()
p = Plan(3, 32, 4)
out = {}
for path in (2, 6):
    p.set_path(path)
    q = p.collide(f)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.collide(f, q)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[path] = q.cpu().numpy()
    p.profile(True)
    p.collide(f, q)
    prof = {k: round(v[0], 4) for k, v in p.profile_read().items() if v[1]}
    p.profile(False)
    print(f"path {path}: {min(ts):.4f} ms per call of {cells} cell(s); kernels {prof}")
print("max |Q6 - Q2| / max |Q2| =", float(np.abs(out[6] - out[2]).max() / np.abs(out[2]).max()))
