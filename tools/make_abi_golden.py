"""Write the golden files of the C ABI test (tests/c_abi/abi_check.c):
tests/golden/abi_<cfg>_f.bin (the seeded input, dvm_inputs) and
tests/golden/abi_<cfg>_q.bin (Q from the direct-sum CPU oracle, oracle/ only),
raw little-endian float64, for c1 (2D, N = 16) and c4 (3D, N = 32).
No CUDA path is involved.  Usage: python tools/make_abi_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dvm_inputs  # noqa: E402
from oracle import oracle  # noqa: E402

for name in ("c1", "c4"):
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)[0]
    Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
    q, _, _ = oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, diagnostics=False)
    out = os.path.join(ROOT, "tests", "golden")
    f.astype("<f8").tofile(os.path.join(out, f"abi_{name}_f.bin"))
    q[0].astype("<f8").tofile(os.path.join(out, f"abi_{name}_q.bin"))
    print(name, cfg.d, cfg.N, cfg.Nbar, Nt, float(np.abs(q).max()))
