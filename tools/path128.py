"""2D v1 sweeps (path 1) vs direction-pair kernels (path 2) per evaluation at N >= 128
(auto-path threshold).  python tools/path128.py"""
import sys, torch, numpy as np; sys.path.insert(0,'.')
from paper_1201_3986_b200 import Plan
for N, nb in ((128, 10), (128, 14), (128, 20), (256, 4), (256, 8), (256, 12)):
    f = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, (1, N * N))).cuda()
    p = Plan(2, N, nb); q = torch.empty_like(f)
    res = []
    for path in (1, 2):
        p.set_path(path)
        for _ in range(3): p.collide(f, q)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30): p.collide(f, q)
        b.record(); torch.cuda.synchronize(); res.append(f"path {path}: {a.elapsed_time(b) / 30 * 1e3:.1f} us")
    print(N, nb, ", ".join(res))
