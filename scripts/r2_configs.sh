#!/bin/bash
# bench lines (both strategies, roofline of the dominant kernel) for every BASELINE config grid
mkdir -p gpurun_out/configs
for c in cube_32 cube_64 cube_128 head_2mm head_1mm_pwc duke_head; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-solve \
    > gpurun_out/configs/$c.json 2> gpurun_out/configs/$c.err; echo $c=$?
done
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
for c in cube_64 cube_128 head_2mm duke_head; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/configs/launches_$c.csv $Q --config $c > /dev/null 2>&1; echo ncu_$c=$?
done
