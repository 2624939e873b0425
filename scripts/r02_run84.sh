#!/bin/bash
# conv2 BackwardFilter through algorithm 8: sub-tiles / pairs / stage width
S="256,64,27,27,192,5,5,2,1"
for t in "" "bfn_msub=2" "bfn_px=64" "bfn_msub=2,bfn_px=64" "bfn2=1" "bfn_stages=4" "bfn_waves=2"; do
  echo "== $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $S --ops 2 --algos 8 --batches 128,64
done
