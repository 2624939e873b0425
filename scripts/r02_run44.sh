#!/bin/bash
for t in "" "fct_epi=8" "fct_epi=4"; do
for sp in "2 3 31 31 16 11 11 2 4" "2 3 36 36 70 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 224 224 64 7 7 3 2" "3 4 30 30 24 5 5 2 2"; do
  UCUDNN_TUNE=$t timeout 60 python scripts/one_small.py $sp 0 0 2>&1 | grep -E "exact|rror" | sed "s/^/[$t] /"
done
UCUDNN_TUNE=$t timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 0 --algos 0 --batches 256,64
done
