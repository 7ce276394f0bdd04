#!/bin/bash
# c5 throughput vs number of cell groups in flight (L2 working-set experiment)
for g in ${GROUPS_LIST:-9 8 7 6}; do
  echo "groups=$g $(DVM_G3_GROUPS=$g python bench.py --cells ${CELLS:-72} --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"])')"
done
