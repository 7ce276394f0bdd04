#!/bin/bash
# Timing split of the cluster kernel (results are wrong with debug bits set).
for dbg in 0 1 2 3; do
  echo "DVM_C3_DEBUG=$dbg"
  DVM_C3_DEBUG=$dbg python bench.py --cells 64 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(' ms/step', d['ms_per_step'], 'cells/s', d['value'])"
done
