#!/bin/bash
# A/B timing of alternative library builds (VIE_LIB_PATH); results are timing only
mkdir -p gpurun_out
for L in "$@"; do
  VIE_LIB_PATH=$PWD/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "$L rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print(d['ms_per_step'], d['stage_ms'])"
done
