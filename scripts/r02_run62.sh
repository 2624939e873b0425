#!/bin/bash
for sp in "2 64 56 56 64 3 3 1 1" "3 64 12 12 64 3 3 1 1" "3 96 8 8 64 5 5 2 1" "2 3 224 224 64 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 31 31 16 11 11 2 4" "4 3 48 48 64 7 7 3 2"; do
  timeout 60 python scripts/one_small.py $sp 2 6 2>&1 | grep -E "exact|rror"
done
timeout 200 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 256,3,224,224,64,7,7,3,2 256,3,227,227,64,11,11,0,4 --ops 2 --algos 6 --batches 256,64
