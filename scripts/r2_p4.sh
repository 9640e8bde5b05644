#!/bin/bash
# pencil4 check: parity subset, bench A/B (pencil4 vs pencil3), phase split of both
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q -x 2>&1 | tail -5
Q="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
timeout 300 $Q > gpurun_out/p4.json 2> gpurun_out/p4.err; echo p4=$?
VIE_NO_PENCIL4=1 timeout 300 $Q > gpurun_out/p3.json 2> gpurun_out/p3.err; echo p3=$?
VIE_P4_PF=-1 timeout 300 $Q > gpurun_out/p4pf.json 2> gpurun_out/p4pf.err; echo p4pf=$?
for f in p4 p3 p4pf; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['ms_per_step'],3), d['stage_ms'])"; done
timeout 300 python scripts/pencil_phases34.py head_1mm 4 2>&1 | tail -10

