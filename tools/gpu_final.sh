#!/bin/bash
# End-of-round measurement pass on one B200 (output: gpurun_out/fin/): the fp64 /
# shared / L2 / HBM microbenchmark, the full GPU suite, bench lines for every
# workload and the reference arm, the ncu launch list of the c5 bench, the ncu
# metrics of the k_fg2 launch in bench.py's configuration (512 cells) and one
# --set full capture of an 18-cell k_fg2 launch (each ncu command only after
# the same command exited 0 without ncu).
set -u
O=gpurun_out/fin
mkdir -p $O
nproc > $O/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench.cu -o /tmp/microbench && \
  timeout 120 /tmp/microbench > $O/microbench.jsonl 2>&1; echo "microbench rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests -q -x -m gpu > $O/gputest.log 2>&1; echo "tests rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 rc=$?" >> $O/status.txt
for w in c1 c2 c3 c4; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
timeout 300 python tools/fg_one.py 512 > $O/plain_one512.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:k_fg2 -c 1 --csv --log-file $O/fg2_bench_launch_metrics.csv python tools/fg_one.py 512 > $O/ncu_metrics.log 2>&1
echo "ncu metrics rc=$?" >> $O/status.txt
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/plain_launches.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $O/status.txt
timeout 300 python tools/fg_one.py 18 > $O/plain_one18.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fg2 -c 1 -o $O/fg2_full18 \
  python tools/fg_one.py 18 > $O/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $O/status.txt
cat $O/status.txt
