#!/bin/bash
# round-2 measurement: bench (both arms), launch list of the headline and of the loop strategy
mkdir -p gpurun_out
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
$Q > gpurun_out/plain.json 2> gpurun_out/plain.err && \
 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $Q > /dev/null 2>&1; echo ncu1=$?
VIE_STRATEGY=loop timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_loop.csv $Q --strategy hosvd_loop > /dev/null 2>&1; echo ncu2=$?
