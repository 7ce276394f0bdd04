#!/bin/bash
# ncu metrics (duration, DRAM bytes, fp64 pipe, l1tex) of every kernel of ONE
# evaluation of c1..c4 as bench.py runs it (plan built and warmed up first; the
# measured call sits between cudaProfilerStart/Stop, ncu --profile-from-start off).
# Output: gpurun_out/ncu_<cfg>.csv; summarise with tools/ncu_config_metrics.py.
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
torch.cuda.profiler.start()
p.collide(f, q)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
PY
mkdir -p gpurun_out
for c in c1 c2 c3 c4; do
  python /tmp/one_eval.py $c > /dev/null 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file gpurun_out/ncu_${c}.csv python /tmp/one_eval.py $c > /dev/null 2>&1
  echo "$c rc=$?"
done
