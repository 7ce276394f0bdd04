#!/bin/bash
# fg_chunks sweep of the c5 kernel over batch sizes (A/B timing only): tools/sweep_chunks.sh "CELLS..." "CHUNKS..." [REPS]
mkdir -p gpurun_out/sweep
for n in $1; do
  for c in $2; do echo -n "cells=$n fg_chunks=$c: "; TUNE="fg_chunks=$c" ORACLE=0 REPS=${3:-2} timeout 300 python tools/fg2_check.py $n | head -1; done
done
