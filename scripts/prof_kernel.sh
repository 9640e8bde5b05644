# usage: bash scripts/prof_kernel.sh <regex> <config> <out>
CMD="python bench.py --config $2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pk.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$1" -s 1 -c 1 -o gpurun_out/$3 $CMD > gpurun_out/ncu_pk.log 2>&1; echo ncu=$?
