#!/bin/bash
# c3 device time per evaluation under env variations ("-" = none)
for spec in "$@"; do
  [ "$spec" = "-" ] && spec=""
  echo -n "== $spec: "
  env $spec python - <<'PY'
import sys, torch; sys.path.insert(0,'.')
import dvm_inputs
from paper_1201_3986_b200 import Plan
cfg=dvm_inputs.CONFIGS['c3']; f=torch.from_numpy(dvm_inputs.make('c3')).cuda()
p=Plan(2,cfg.N,cfg.Nbar); q=torch.empty_like(f)
for _ in range(5): p.collide(f,q)
torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): p.collide(f,q)
b.record(); torch.cuda.synchronize(); print(f"{a.elapsed_time(b)/50*1e3:.1f} us per evaluation")
PY
done
