#!/bin/bash
# ncu metrics (duration, DRAM bytes, fp64 pipe, l1tex) for every kernel of one evaluation of c1..c4
cat > /tmp/one_eval.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, dvm_inputs
from paper_1201_3986_b200 import Plan
name = sys.argv[1]
cfg = dvm_inputs.CONFIGS[name]
f = torch.from_numpy(dvm_inputs.make(name)).cuda()
p = Plan(cfg.d, cfg.N, cfg.Nbar)
q = torch.empty_like(f)
for _ in range(3): p.collide(f, q)
torch.cuda.synchronize()
p.collide(f, q)
torch.cuda.synchronize()
PY
for c in c1 c2 c3 c4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file gpurun_out/ncu_${c}.csv python /tmp/one_eval.py $c > /dev/null 2>&1
  echo "$c rc=$?"
done
