#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
Q="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
for c in head_1mm cube_64; do
timeout 300 $Q --config $c > gpurun_out/q.json 2> gpurun_out/q.err
python -c "
import json; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), d['stage_ms'], {k: round(v.get('ms_per_step',0),3) for k, v in d['strategies'].items()})"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_decomp_z -c 1 $Q 2>&1 | grep duration
