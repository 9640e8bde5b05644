#!/bin/bash
# round-2 evidence run (v4, v5, ...: EVID): GPU tests, smoke, bench (both arms), launch lists (both strategies),
# ncu --set full of each hot kernel summarised ON THE BOX (the .ncu-rep files are deleted so
# gpurun_out stays under the copy-back limit), config lines, pencil phase profile.
O=gpurun_out/${EVID:-v5}
mkdir -p $O/configs
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > $O/gputests.txt; cat $O/gputests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
Q="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-solve"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $Q > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_loop.csv $Q --strategy hosvd_loop > /dev/null 2>&1; echo ncu2=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pencil4|k_decomp_s_mma|k_col_fwd2|k_row_fwd2|k_col_inv2|k_row_inv2" -s 6 -c 6 -o /tmp/full_decompress $Q > $O/ncu_full.log 2>&1; echo ncu3=$?
python profiles/ncu_extract.py /tmp/full_decompress.ncu-rep > $O/ncu_full_decompress.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 1 -c 1 -o /tmp/full_loop $Q --strategy hosvd_loop > $O/ncu_full_loop.log 2>&1; echo ncu4=$?
python profiles/ncu_extract.py /tmp/full_loop.ncu-rep > $O/ncu_full_loop.txt 2>&1
for c in cube_32 cube_64 cube_128 head_2mm head_1mm_pwc duke_head; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-solve \
    > $O/configs/$c.json 2> $O/configs/$c.err; echo $c=$?
done
for c in cube_64 cube_128 head_2mm duke_head; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/configs/launches_$c.csv $Q --config $c > /dev/null 2>&1; echo ncu_$c=$?
done
if [ -f gpurun_prof.so ]; then
  PROF_SO=$PWD/gpurun_prof.so timeout 600 python scripts/pencil_phases34.py head_1mm 4 > $O/pencil4_phases.txt 2>&1; echo phases=$?
fi
du -sh $O
