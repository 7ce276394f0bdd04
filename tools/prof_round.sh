#!/bin/bash
# GPU tests, default bench, launch list and one --set full capture of k_fgain3d (18 cells)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
CMD="python bench.py --cells 18 --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_cur.csv $CMD > gpurun_out/ncu_launch_cur.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fgain3d -s 1 -c 1 -o gpurun_out/prof_cur $CMD > gpurun_out/ncu_full_cur.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_fgain3d -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/traffic_bench.csv 2>&1
echo done
