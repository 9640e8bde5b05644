#!/bin/bash
# A/B timing over values of one environment variable: ab_env.sh VAR v1 v2 ...
mkdir -p gpurun_out
VAR=$1; shift
for V in "$@"; do
  env $VAR=$V timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "$VAR=$V rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print(d['ms_per_step'], d['stage_ms'])"
done
