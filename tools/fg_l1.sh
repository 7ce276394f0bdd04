#!/bin/bash
# L1 hit rate and shared-memory configuration of k_fgain3d for given builds
for n in "$@"; do
  echo "== $n"
  DVM_LIB=tools/ab/libdvm_$n.so PATHS=4 REPS=1 ncu --metrics l1tex__t_sector_hit_rate.pct,launch__shared_mem_config_size,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum,gpu__time_duration.sum --clock-control none -k regex:k_fgain3d -s 1 -c 1 --csv python tools/fg_check.py 8 18 2>/dev/null | grep -E "hit_rate|config_size|lookup|duration" | awk -F'","' '{print $(NF-2), $NF}'
done
