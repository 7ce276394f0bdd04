"""c5 cells through the 3D N = 64 kernel (k_fg2): per-evaluation time (CUDA
events, min / median of REPS), optionally the phase timings (timing_dbg bits:
1 phase A only, 2 phase B only, 4 no taps; Q wrong there), and oracle parity on
sampled nodes of the last cell.  Usage: python tools/fg2_check.py CELLS [DBG...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 18
dbgs = [int(x) for x in sys.argv[2:]]
reps = int(os.environ.get("REPS", "4"))
f = torch.from_numpy(dvm_inputs.make("c5", cells=cells)).cuda()
p = Plan(3, 64, 8)
for kv in os.environ.get("TUNE", "").split():
    k, v = kv.split("=")
    p.set_tuning(k, int(v))


def timed(p):
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
    return q, ts


q, ts = timed(p)
q = q.cpu().numpy()
print(f"k_fg2: min {ts[0]:.2f} ms, median {ts[len(ts) // 2]:.2f} ms for {cells} cells "
      f"-> {cells / ts[0] * 1e3:.1f} cells/s", flush=True)
for dbg in dbgs:
    p.set_tuning("timing_dbg", dbg)
    _, tsd = timed(p)
    print(f"   timing_dbg {dbg}: min {tsd[0]:.2f} ms", flush=True)
p.set_tuning("timing_dbg", 0)
if os.environ.get("ORACLE", "1") == "1":
    from oracle import oracle
    fc = dvm_inputs.make("c5", cells=cells)[cells - 1]
    pts = np.arange(0, 64 ** 3, 64 ** 3 // 97)
    qo, _, _ = oracle.collide(fc, 3, 64, 8, p.Ntilde, 8.0, points=pts, diagnostics=False)
    rel = np.abs(q[cells - 1][pts] - qo[0]).max() / np.abs(qo[0]).max()
    print(f"oracle parity (cell {cells - 1}, {len(pts)} nodes): {rel:.3e}")
