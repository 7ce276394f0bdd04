"""One c5 evaluation of CELLS cells (for ncu captures), optionally with timing_dbg bits.
Usage: python tools/fg_one.py CELLS [TIMING_DBG]"""
import sys

import torch

sys.path.insert(0, ".")
import dvm_inputs  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 18
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
f = torch.from_numpy(dvm_inputs.make("c5", cells=cells)).cuda()
p = Plan(3, 64, 8)
p.set_tuning("timing_dbg", dbg)
q = p.collide(f)
torch.cuda.synchronize()
print("ok", float(q.abs().max()))
