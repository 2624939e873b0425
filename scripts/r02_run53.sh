#!/bin/bash
for op in 0 1; do
for sp in "2 64 27 27 192 5 5 2 1" "3 64 12 12 64 3 3 1 1" "2 32 16 16 48 3 3 1 1" "2 64 28 28 128 3 3 1 1" "2 192 13 13 64 3 3 1 1" "1 64 56 56 64 3 3 1 1" "2 32 9 11 40 5 5 2 1" "2 96 7 7 256 3 3 0 1"; do
  timeout 60 python scripts/one_small.py $sp $op 7 2>&1 | grep -E "exact|rror|trace"
done
done
timeout 60 python scripts/one_small.py 2 64 27 27 192 5 5 2 1 0 0 2>&1 | grep -E "exact|rror|trace"
timeout 200 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 --ops 0,1 --algos 0,5,7 --batches 256,128,64
