"""c2 (d=2, N=64, N̄=8): 100 explicit Euler steps, dt = 0.01 (reading R11), and
the same with TVD-RK2: mass, momentum and energy drift relative to step 0
(mass at round-off, momentum/energy aliasing-limited)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

f0 = dvm_inputs.make("c2")[0]
p = Plan(2, 64, 8)
for method in ("euler", "rk2"):
    f = torch.from_numpy(f0.copy()).cuda()
    m = getattr(p, method)(f, 0.01, 100)
    m0 = m[0]
    out = {"method": method, "steps": 100, "dt": 0.01,
           "mass_rel_drift": float(abs(m[-1, 0] - m0[0]) / m0[0]),
           "momentum_drift": [float(m[-1, 1] - m0[1]), float(m[-1, 2] - m0[2])],
           "energy_rel_drift": float(abs(m[-1, 3] - m0[3]) / m0[3]),
           "min_f": float(f.min().item())}
    print(json.dumps(out))
