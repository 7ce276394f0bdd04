#!/bin/bash
# A/B of k_fg2 variants (tools/ab/libdvm_<name>.so) on CELLS c5 cells, interleaved rounds.
# Usage: tools/ab_fg2.sh CELLS ROUNDS name...   (output: one line per variant and round)
CELLS=$1; ROUNDS=$2; shift 2
for r in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    echo -n "$v r$r: "
    DVM_LIB=tools/ab/libdvm_$v.so ORACLE=${ORACLE:-0} REPS=${REPS:-4} timeout 300 python tools/fg2_check.py $CELLS | tr '\n' ' '
    echo
  done
done
