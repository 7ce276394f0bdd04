#!/bin/bash
# k_fgain3d phase timing: DVM_FG_DEBUG bit sets (1 no B work, 2 no A work, 4 no taps, 8 no T2D copy)
for dbg in ${DBGS:-0 1 2 4 8 3}; do
  echo "dbg=$dbg"
  DVM_FG_DEBUG=$dbg timeout 300 python tools/fg_check.py ${NBAR:-8} ${CELLS:-18} 2>&1 | grep "path 4"
done
