import sys, torch
sys.path.insert(0, ".")
import dvm_inputs
from paper_1201_3986_b200 import Plan
f = torch.from_numpy(dvm_inputs.make("c5", cells=2)).cuda()
p = Plan(3, 64, 1)
p.set_path(4)
q = p.collide(f)
torch.cuda.synchronize()
print("ok", float(q.abs().max()))
