#!/bin/bash
for t in "" "slice_cap_kib=50000" "slice_cap_kib=60000" "slice_cap_kib=62000"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 200 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 --ops 1 --algos 7 --batches 256,128 2>&1 | grep -v "^256"
done
