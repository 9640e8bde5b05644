#!/bin/bash
# repetition sweep of small matvecs against the oracle (intermittent-ordering probe)
O=gpurun_out/flake3; mkdir -p $O
for c in "4 5 200 25 100 hosvd_decompress" "4 5 200 25 100 hosvd_loop" "5 6 32 25 100 hosvd_loop" \
         "6 7 64 20 100 hosvd_decompress" "6 7 64 20 100 hosvd_loop" "3 4 125 25 100 hosvd_decompress" \
         "8 6 100 12 100 hosvd_decompress 1 1" "8 6 100 12 100 hosvd_loop 1 1" "9 8 128 25 100 hosvd_decompress" \
         "10 9 96 8 100 hosvd_decompress 0 0" "7 5 120 6 100 hosvd_decompress 1 0" "70 9 32 4 60 hosvd_loop"; do
  timeout 300 python scripts/flake_probe.py $c 2>/dev/null | tail -1 >> $O/out.txt
done
cat $O/out.txt
