"""c3 (2D, N = 256, N̄ = 16): per-evaluation time of the line-walk pair kernels
(path 2) and the tile kernel (path 7), CUDA events, min of 20, per-kernel
profile and agreement.  Usage: python tools/c3_paths.py [NAME]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = dvm_inputs.CONFIGS[name]
f = torch.from_numpy(dvm_inputs.make(name)).cuda()
p = Plan(cfg.d, cfg.N, cfg.Nbar)
out = {}
for path in (2, 7):
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
    print(f"{name} path {path}: {min(ts):.4f} ms; kernels {prof}")
print("max |Q7 - Q2| / max |Q2| =", float(np.abs(out[7] - out[2]).max() / np.abs(out[2]).max()))
