#!/bin/bash
# sub-phase timing of k_gain3d: DVM_G3_DEBUG bits: 1 skip A, 2 skip B, 4 skip A3 (T), 8 skip A1 (gather+scan)
for dbg in ${DBGS:-2 6 10 14 3}; do
  echo "dbg=$dbg $(DVM_G3_DEBUG=$dbg python bench.py --cells ${CELLS:-36} --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"])')"
done
