#!/bin/bash
# parity tests + one short bench (stage times) -- the inner build/measure loop
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -6
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/quick.json 2> gpurun_out/quick.err
echo "bench rc=$?"; tail -3 gpurun_out/quick.err
python -c "
import json; d=json.load(open('gpurun_out/quick.json')); print(d['ms_per_step'], d['stage_ms'])"
