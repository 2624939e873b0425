#!/bin/bash
# conv1 BackwardFilter (fct_bwdf) ring depth sweep
A="256,3,224,224,64,11,11,2,4"; R="256,3,224,224,64,7,7,3,2"
for r in 0 9 10 12 14 16 20; do echo "== R ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_bf_ring=$r) timeout 300 python scripts/time_table.py $R --ops 2 --algos 6 --batches 256; done
for r in 0 15 18 20 24 28; do echo "== A ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_bf_ring=$r) timeout 300 python scripts/time_table.py $A --ops 2 --algos 6 --batches 256; done
