#!/bin/bash
for t in "" "fct_bd_pair=0"; do
for sp in "2 3 31 31 16 11 11 2 4" "3 3 227 227 64 11 11 0 4" "3 4 30 30 24 5 5 2 2" "5 3 63 63 20 11 11 1 4" "2 1 20 20 5 3 3 1 2" "2 3 36 36 64 7 7 3 2" "3 3 47 51 64 11 11 2 4" "2 3 224 224 64 7 7 3 2" "1 3 224 224 64 7 7 3 2" "2 3 100 140 32 7 7 3 2" "1 3 45 45 8 11 11 0 4"; do
  UCUDNN_TUNE=$t timeout 60 python scripts/one_small.py $sp 1 0 2>&1 | grep -E "exact|rror" | sed "s/^/[$t] /"
done
UCUDNN_TUNE=$t timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 1 --algos 0 --batches 256,64
done
