#!/bin/bash
# c5 bench under env variations: each arg "VAR=val ..." ("-" = none)
for spec in "$@"; do
  [ "$spec" = "-" ] && spec=""
  echo "== $spec"
  env $spec timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'])"
done
