#!/bin/bash
# quick correctness + timing loop for gain3d changes (one gpurun call)
timeout 600 python -m pytest tests -m gpu -q -x -k "gain3d or c4 or c5 or constant or determinism or full_small" > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?" ; tail -2 gpurun_out/q_tests.log
for dbg in ${DBGS:-0 2}; do
  echo "dbg=$dbg $(DVM_G3_DEBUG=$dbg timeout 300 python bench.py --cells ${CELLS:-36} --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), d["ms_per_step"])')"
done
