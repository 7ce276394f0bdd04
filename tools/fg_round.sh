#!/bin/bash
# k_fgain3d: phase timing (DVM_FG_DEBUG bits), ncu launch list, one --set full capture.
mkdir -p gpurun_out
TAG=${TAG:-fg}
DBGS=${DBGS:-"0 1 2 4 3"} CELLS=${CELLS:-18} bash tools/fg_phase.sh > gpurun_out/phase_${TAG}.log 2>&1
CMD="python bench.py --cells ${CELLS:-18} --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
[ -n "$NOFULL" ] && exit 0
ncu --set full --clock-control none --import-source on -k regex:k_fgain3d -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu-done
