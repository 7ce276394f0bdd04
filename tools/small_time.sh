#!/bin/bash
# c1 / c2 device time per evaluation for several builds (tools/ab/libdvm_<name>.so)
for n in "$@"; do echo -n "$n: "; DVM_LIB=tools/ab/libdvm_$n.so python - <<'PY'
import sys, torch; sys.path.insert(0,'.')
import dvm_inputs
from paper_1201_3986_b200 import Plan
out=[]
for name in ("c1","c2"):
    cfg=dvm_inputs.CONFIGS[name]; f=torch.from_numpy(dvm_inputs.make(name)).cuda()
    p=Plan(2,cfg.N,cfg.Nbar); q=torch.empty_like(f)
    for _ in range(5): p.collide(f,q)
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100): p.collide(f,q)
    b.record(); torch.cuda.synchronize(); out.append(f"{name} {a.elapsed_time(b)/100*1e3:.1f} us")
print(", ".join(out))
PY
done
