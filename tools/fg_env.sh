#!/bin/bash
# k_fgain3d timing under env variations: each arg is "VAR=val VAR2=val" (quoted); "-" = none
mkdir -p gpurun_out
for spec in "$@"; do
  [ "$spec" = "-" ] && spec=""
  echo "== $spec"
  env $spec PATHS=4 timeout 300 python tools/fg_check.py ${NBAR:-8} ${CELLS:-18} 2>&1 | grep "path 4"
done
