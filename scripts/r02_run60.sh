#!/bin/bash
for t in "" "fct_bf_dtma=0"; do
for sp in "2 3 36 36 64 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 224 224 64 7 7 3 2" "4 3 48 48 64 7 7 3 2" "2 1 20 20 16 3 3 1 2" "3 4 30 30 32 5 5 2 2"; do
  UCUDNN_TUNE=$t timeout 60 python scripts/one_small.py $sp 2 6 2>&1 | grep -E "exact|rror|trace" | sed "s/^/[$t] /"
done
UCUDNN_TUNE=$t timeout 120 python scripts/time_table.py 256,3,224,224,64,7,7,3,2 256,3,227,227,64,11,11,0,4 --ops 2 --algos 6 --batches 256,64
done
