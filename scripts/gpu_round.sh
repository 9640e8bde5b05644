#!/bin/bash
# One GPU session per phase (one ncu tool per gpurun call):
#   bash scripts/gpu_round.sh main  -- tests, bench (both arms), ncu launch list
#   bash scripts/gpu_round.sh full  -- ncu --set full capture of the top kernels
set -o pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
if [ "${1:-main}" = main ]; then
  timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
  timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
  $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1; echo ncu1=$?
else
  $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
  ncu --set full --clock-control none --import-source on -k regex:"k_pencil2|k_decomp_s_mma|k_col_fwd2|k_row_fwd2|k_col_inv2|k_row_inv2" -s 10 -c 6 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
