#!/bin/bash
for sp in "2 64 56 56 64 3 3 1 1" "3 64 12 12 64 3 3 1 1" "2 32 16 16 48 3 3 1 1" "2 128 28 28 128 3 3 1 1" "3 96 8 8 64 5 5 2 1" "2 64 20 24 32 3 3 0 1" "1 256 8 8 128 3 3 1 1"; do
  timeout 60 python scripts/one_small.py $sp 2 6 2>&1 | grep -E "exact|rror|trace"
done
timeout 120 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 --ops 2 --algos 6,8 --batches 256,128,64
