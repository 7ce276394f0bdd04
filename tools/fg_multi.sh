#!/bin/bash
# k_fgain3d timing (18 cells) for several builds: tools/fg_multi.sh name1 name2 ... (tools/ab/libdvm_<name>.so)
for i in 1 2; do
  for n in "$@"; do
    echo -n "$n: "; DVM_LIB=tools/ab/libdvm_$n.so PATHS=4 timeout 300 python tools/fg_check.py 8 ${CELLS:-18} | grep "path 4"
  done
done
