#!/bin/bash
# A/B timing of k_fgain3d: tools/ab/libdvm_old.so vs the in-tree build, alternating
mkdir -p gpurun_out
for i in 1 2; do
  echo "old:"; DVM_LIB=tools/ab/libdvm_old.so PATHS=4 timeout 300 python tools/fg_check.py 8 ${CELLS:-18} | grep "path 4"
  echo "new:"; PATHS=4 timeout 300 python tools/fg_check.py 8 ${CELLS:-18} | grep "path 4"
done
