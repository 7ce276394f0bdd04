import sys, time, os
sys.path.insert(0, "/root/repo")
import torch, dvm_inputs
from paper_1201_3986_b200 import Plan
for name, d, N, Nb in (("c1", 2, 16, 4), ("c2", 2, 64, 8), ("c3", 2, 256, 16)):
    f0 = torch.from_numpy(dvm_inputs.make(name)[0].copy()).cuda()
    p = Plan(d, N, Nb)
    for path in (0, 1):
        p.set_path(path)
        q = torch.empty_like(f0)
        for _ in range(3): p.collide(f0, q)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(50): p.collide(f0, q)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        f = f0.clone(); p.euler(f, 0.01, 5, moments=False)
        f = f0.clone(); torch.cuda.synchronize(); t2 = time.perf_counter()
        p.euler(f, 0.01, 100, moments=False); t3 = time.perf_counter()
        print(name, "path", path, "collide us %.1f" % ((t1-t0)/50*1e6), "euler100 ms %.2f" % ((t3-t2)*1e3), flush=True)
