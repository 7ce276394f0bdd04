#!/bin/bash
# one --set full capture of k_fgain3d under DVM_FG_DEBUG=$DBG (tag $TAG)
mkdir -p gpurun_out
CMD="python tools/fg_check.py 8 ${CELLS:-18}"
DVM_FG_DEBUG=${DBG:-0} PATHS=4 ncu --set full --clock-control none --import-source on -k regex:k_fgain3d -s 1 -c 1 \
    -o gpurun_out/prof_${TAG:-dbg} $CMD > gpurun_out/ncu_${TAG:-dbg}.log 2>&1
echo done
