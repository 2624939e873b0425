#!/bin/bash
L="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1 256,64,56,56,192,3,3,1,1"
for t in "" "two_sm_min_bn=64" "two_sm_min_bn=64,pc2_ksub=1"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5,7 --batches 256,64 2>&1
done
