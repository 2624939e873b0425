#!/bin/bash
# AlexNet conv2 / conv4 Forward: CTA-pair stage / sub-tile knobs, and the 1-SM kernel
for t in "" "pc2_ksub=1" "pc2_msub=2" "two_sm=0"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 --ops 0 --algos 5 --batches 256 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,384,13,13,256,3,3,1,1 --ops 0 --algos 5 --batches 128 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,192,13,13,384,3,3,1,1 --ops 0 --algos 5 --batches 256 | grep algo
done
