#!/bin/bash
for sp in "2 3 31 31 16 11 11 2 4" "2 3 36 36 70 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 224 224 64 7 7 3 2" "1 2 40 40 8 11 11 0 4" "3 4 30 30 24 5 5 2 2" "5 3 63 63 20 11 11 1 4" "4 3 48 48 64 7 7 3 2"; do
  timeout 60 python scripts/one_small.py $sp 0 0 2>&1 | grep -E "exact|rror"
done
timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 0 --algos 0 --batches 256,64
