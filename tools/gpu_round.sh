#!/bin/bash
# One GPU session: bench, ncu launch list, a full capture of the top kernel, and PCIe/DRAM counters.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run_copy -s 5 -c 2 -o gpurun_out/prof_$TAG -f python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__write_bytes.sum,pcie__read_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,syslts__t_bytes.sum --clock-control none -k regex:k_run_copy -s 5 -c 5 --csv --log-file gpurun_out/io_$TAG.csv python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_io_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log gpurun_out/ncu_io_$TAG.log
