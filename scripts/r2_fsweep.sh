#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "loop" 2>&1 | tail -2
Q="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
for cfg in "4 4" "6 4" "6 6" "6 8" "8 4"; do
  set -- $cfg
  VIE_STRATEGY=loop VIE_FUSED_LA=$1 VIE_FUSED_CG=$2 timeout 300 $Q > gpurun_out/fs.json 2> gpurun_out/fs.err
  python -c "
import json; d=json.load(open('gpurun_out/fs.json')); print('LA=$1 CG=$2', round(d['ms_per_step'],3), d['stage_ms']['pencil'])"
done
