#!/bin/bash
# One GPU call: plain run, then the ncu launch list and one full capture of the
# dominant kernel (the guide's recipe).  Usage: tools/ncu_round.sh <tag> <kernel-regex>
set -x
TAG=${1:-r01}
KREG=${2:-k_rowsum}
CMD="python bench.py --cells ${CELLS:-14} --steps 1 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
$CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREG} -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu-done
