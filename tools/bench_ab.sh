#!/bin/bash
# A/B of the c5 bench (full batch): tools/ab/libdvm_old.so vs the in-tree build
for i in 1 2; do
  echo "old:"; DVM_LIB=tools/ab/libdvm_old.so timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'])"
  echo "new:"; timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'])"
done
