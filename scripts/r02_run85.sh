#!/bin/bash
# algorithm 8 BackwardFilter: 1-SM vs CTA-pair tiles across the AlexNet / ResNet layers
S="256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1 256,256,14,14,256,3,3,1,1 256,512,7,7,512,3,3,1,1 256,128,28,28,128,3,3,1,1"
for t in "" "bfn2=1" "bfn2=0"; do
  echo "== $t"; UCUDNN_TUNE=$t timeout 600 python scripts/time_table.py $S --ops 2 --algos 8 --batches 256,128,64
done
