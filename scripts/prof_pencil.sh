CMD="python bench.py --config head_2mm --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pp.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_pencil" -s 1 -c 1 -o gpurun_out/prof_pen $CMD > gpurun_out/ncu_pen.log 2>&1; echo ncu=$?
