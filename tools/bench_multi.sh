#!/bin/bash
# c5 bench for several "lib:ENV=val" specs (lib = tools/ab/libdvm_<lib>.so, "-" = in-tree)
for i in 1 2; do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
    L=""; [ "$lib" != "-" ] && L="DVM_LIB=tools/ab/libdvm_$lib.so"
    echo -n "$spec: "
    env $L $envs timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value'],1), round(d['ms_per_step'],1))"
  done
done
