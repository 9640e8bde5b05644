#!/bin/bash
mkdir -p gpurun_out
VIE_DECOMP_TILE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
Q="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
VIE_DECOMP_TILE=1 timeout 300 $Q > gpurun_out/dt.json 2> gpurun_out/dt.err; echo dt=$?
timeout 300 $Q > gpurun_out/dm.json 2> gpurun_out/dm.err; echo dm=$?
for f in dt dm; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['ms_per_step'],3), d['stage_ms'])"; done
