#!/bin/bash
run() { python bench.py --cells ${CELLS:-144} --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(' ms/step', round(d['ms_per_step'],1), 'cells/s', round(d['value'],2))"; }
echo "cluster mode"; DVM_C3_MODE=cluster run
for g in 7 8 9; do echo "soft groups=$g"; DVM_C3_GROUPS=$g run; done
