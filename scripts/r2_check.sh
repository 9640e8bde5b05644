#!/bin/bash
# post-change check: GPU tests, determinism + oracle repeat probes, bench, slab bench (N > 1 code path on one GPU)
O=gpurun_out/${EVID:-chk}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > $O/gputests.txt; cat $O/gputests.txt
timeout 900 python scripts/determinism_probe.py 4 5 200 25 600 2>&1 | grep -v Warn > $O/determinism.txt
timeout 300 python scripts/flake_probe.py 4 5 200 25 300 2>/dev/null | tail -1 >> $O/determinism.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-solve > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 600 python bench.py --slab --steps 5 --warmup 3 --no-cpu-baseline --no-solve > $O/slab.json 2> $O/slab.err; echo slab=$?
