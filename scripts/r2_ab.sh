#!/bin/bash
# quick A/B of the current library: parity of the pencil paths + head_1mm bench (3 runs)
O=gpurun_out/ab
mkdir -p $O
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-solve > $O/bench_$i.json 2> $O/bench_$i.err; echo bench$i=$?
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_cp.py -m gpu -q -x 2>&1 | tail -4 > $O/tests.txt; cat $O/tests.txt
