#!/bin/bash
L="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1 256,64,28,28,64,3,3,1,1"
for t in "" "strip=1,strip_msub=4" "strip=1,strip_msub=2"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5,7 --batches 256,128,64 2>&1
done
