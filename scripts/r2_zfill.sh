O=gpurun_out/zf2; mkdir -p $O
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
for v in z3 z0 main; do
  if [ $v = main ]; then L=""; else L="VIE_LIB_PATH=$PWD/gpurun_$v.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_decomp_s_mma --csv --log-file $O/dec_$v.csv $Q > /dev/null 2>&1; echo $v=$?
done
VIE_LIB_PATH=$PWD/gpurun_z3.so timeout 300 python scripts/flake_probe.py 4 5 200 25 300 2>/dev/null | tail -1 > $O/flake_z3.txt
VIE_LIB_PATH=$PWD/gpurun_z0.so timeout 300 python scripts/flake_probe.py 4 5 200 25 300 2>/dev/null | tail -1 > $O/flake_z0.txt
