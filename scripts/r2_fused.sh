#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -4
Q="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
timeout 300 $Q > gpurun_out/fu.json 2> gpurun_out/fu.err; echo fu=$?
VIE_NO_FUSED=1 timeout 300 $Q > gpurun_out/nf.json 2> gpurun_out/nf.err; echo nf=$?
for f in fu nf; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['ms_per_step'],3), d['stage_ms'])"; done
tail -3 gpurun_out/fu.err
