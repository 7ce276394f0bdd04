"""Device time of the c2 time loops (100 steps, dt = 0.01) with and without the
CUDA-graph replay, Euler and TVD-RK2, plus a 3D (N = 32) check that the
cooperative gain kernel replays from a graph.  python tools/stepper_times.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

res = {}
for name, d, N, Nb in (("c2", 2, 64, 8), ("c4", 3, 32, 4)):
    f0 = torch.from_numpy(dvm_inputs.make(name)[0].copy()).cuda()
    p = Plan(d, N, Nb)
    for method in ("euler", "rk2"):
        for graphs in (True, False):
            p.set_graphs(graphs)
            f = f0.clone()
            getattr(p, method)(f, 0.01, 5, moments=False)  # warm
            f = f0.clone()
            torch.cuda.synchronize()
            l0 = p.launches()
            t0 = time.perf_counter()
            getattr(p, method)(f, 0.01, 100, moments=True)
            t1 = time.perf_counter()
            res[f"{name}_{method}_{'graph' if graphs else 'direct'}"] = {
                "ms_100_steps": (t1 - t0) * 1e3, "launches": p.launches() - l0}
            print(name, method, graphs, json.dumps(res[f"{name}_{method}_{'graph' if graphs else 'direct'}"]), flush=True)
