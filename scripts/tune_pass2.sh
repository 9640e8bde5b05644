#!/bin/bash
# parity + stage times of the register-staged passes for a few row tile sizes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for L in 0 8 16; do
  VIE_ROW_LINES=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tune_$L.json 2> gpurun_out/tune_$L.err
  echo "rows=$L rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/tune_$L.json')); print(d['ms_per_step'], d['roofline'].get('stage_ms') or d.get('stage_ms') or {k:v for k,v in d.items() if 'stage' in k})"
done
