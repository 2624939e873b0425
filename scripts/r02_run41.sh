#!/bin/bash
for t in "strip=1" "strip=1,strip_msub=1" "sswap=1"; do
for sp in "2 64 27 27 96 5 5 2 1 0 5" "2 64 27 27 96 5 5 2 1 1 5" "3 32 14 14 64 3 3 1 1 0 5" "3 32 14 14 64 3 3 1 1 1 5" "2 192 13 13 64 3 3 1 1 1 5" "5 64 27 27 192 5 5 2 1 1 5" "2 96 11 9 48 3 3 1 1 0 5"; do
  UCUDNN_TUNE=$t timeout 60 python scripts/one_small.py $sp 2>&1 | grep -E "exact|rror" | sed "s/^/$t /"
done
done
L="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1"
for t in "" "strip=1" "strip=1,strip_msub=1"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256,64 2>&1
done
