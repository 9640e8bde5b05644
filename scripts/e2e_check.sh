#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "batch or mixed" 2>&1 | tail -3
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/e2e.json 2> gpurun_out/e2e.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/e2e.json')); print(d['value'], d['e2e'])"
