#!/bin/bash
L="256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1"
for t in "" "pc2_ksub=1" "pc_ksub=1" "pc_ksub=1,pc2_ksub=1"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256,128,64 2>&1
done
