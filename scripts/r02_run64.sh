#!/bin/bash
L="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1"
for t in "" "pc_msub=2" "pc_cps=1" "pc_msub=2,pc_cps=1"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 200 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256,64 2>&1 | grep -v "^256,128,28.*op=F" 
done
