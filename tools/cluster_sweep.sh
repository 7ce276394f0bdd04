#!/bin/bash
for cl in 16 8 4; do
  echo "cluster=$cl"
  DVM_C3_CLUSTER=$cl python bench.py --cells 128 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(' ms/step', d['ms_per_step'], 'cells/s', d['value'])"
done
