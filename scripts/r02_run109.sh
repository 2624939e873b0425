#!/bin/bash
# algorithm 8 with its new CTA-pair default: stage width / count / waves sweep at the planned micro-batches
for t in "" "bfn_px=64" "bfn_stages=6" "bfn_waves=2" "bfn_msub=2"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 --ops 2 --algos 8 --batches 64 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1 --ops 2 --algos 8 --batches 128 | grep algo
done
