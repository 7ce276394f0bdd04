#!/bin/bash
# Phase timing of k_gain3d (DVM_G3_DEBUG bit0 skips phase A, bit1 skips phase B)
# and one ncu --set full capture.  Usage: tools/g3_phase.sh <tag> [cells]
TAG=${1:-g3}
CELLS=${2:-36}
mkdir -p gpurun_out
for dbg in 0 1 2 3; do
  echo "dbg=$dbg $(DVM_G3_DEBUG=$dbg python bench.py --cells $CELLS --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["kernel_profile_ms"])')"
done > gpurun_out/phase_${TAG}.log 2>&1
cat gpurun_out/phase_${TAG}.log
if [ "${NCU:-1}" = "1" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_gain3d -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --cells 9 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu rc=$?
fi
