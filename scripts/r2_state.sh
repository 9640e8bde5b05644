#!/bin/bash
# round-2 state check: bench, pencil3 phase split, launch list, ncu full of the top two kernels, GPU tests
mkdir -p gpurun_out
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python scripts/pencil3_phases.py head_1mm > gpurun_out/phases.txt 2>&1; echo phases=$?
$Q > gpurun_out/plain.json 2> gpurun_out/plain.err && \
 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $Q > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pencil3|k_decomp_s_mma" -s 4 -c 2 -o gpurun_out/full_r2a $Q > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
