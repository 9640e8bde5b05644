#!/bin/bash
# round-2 evidence run: GPU tests, smoke, bench (both arms), launch lists (both strategies),
# one ncu --set full capture of each hot kernel
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final/gputests.txt; cat gpurun_out/final/gputests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo ref=$?
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
$Q > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv $Q > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches_loop.csv $Q --strategy hosvd_loop > /dev/null 2>&1; echo ncu2=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pencil4|k_decomp_s_mma|k_col_fwd2|k_row_fwd2|k_col_inv2|k_row_inv2" -s 6 -c 6 -o gpurun_out/final/full_decompress $Q > gpurun_out/final/ncu_full.log 2>&1; echo ncu3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 1 -c 1 -o gpurun_out/final/full_loop $Q --strategy hosvd_loop > gpurun_out/final/ncu_full_loop.log 2>&1; echo ncu4=$?
