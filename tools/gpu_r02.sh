#!/bin/bash
# Round-2 measurement pass on one B200: new GPU tests, bench lines for every
# workload, the ncu launch list of the c5 bench and one ncu metric capture of
# the k_fg2 launch in bench.py's configuration (512 cells).  Output: gpurun_out/r2/
set -u
O=gpurun_out/r2
mkdir -p $O
nproc > $O/nproc.txt
timeout 600 python -m pytest tests -q -x -m gpu -k "c_caller or shards or levels_abi or smoke" > $O/tests_new.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?" >> $O/status.txt
for w in c1 c2 c3 c4; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
timeout 300 python tools/fg_one.py 512 > $O/plain_one512.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_fg2 -c 1 --csv --log-file $O/fg2_bench_launch_metrics.csv python tools/fg_one.py 512 > $O/ncu_metrics.log 2>&1
echo "ncu metrics rc=$?" >> $O/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $O/status.txt
cat $O/status.txt
