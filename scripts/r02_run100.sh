#!/bin/bash
# stride-1 TMEM-operand BackwardFilter (fct_bwdf1) ring depth sweep on the ResNet 3x3 layers
S="256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1"
for r in 0 4 5 6 8; do echo "== ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_bf1_ring=$r) timeout 300 python scripts/time_table.py $S --ops 2 --algos 6 --batches 256; done
