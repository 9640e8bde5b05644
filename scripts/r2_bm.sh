#!/bin/bash
Q="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-solve --strategy hosvd_loop"
for lib in paper_1811_00484_b200/libvie_b200.so gpurun_bm32.so; do
 for la in 4 6 8; do
  VIE_LIB_PATH=$PWD/$lib VIE_FUSED_LA=$la timeout 300 $Q > gpurun_out/bm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bm.json')); print('$lib LA=$la', round(d['ms_per_step'],3))"
  VIE_LIB_PATH=$PWD/$lib VIE_FUSED_LA=$la timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -s 1 -c 1 $Q 2>&1 | grep dram__
 done
done
