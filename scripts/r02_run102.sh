#!/bin/bash
# conv1 Forward / BackwardData row-ring depth sweep (the BackwardFilter kernels preferred shallow rings)
A="256,3,224,224,64,11,11,2,4"; R="256,3,224,224,64,7,7,3,2"
for r in 0 23 27 31; do echo "== F A ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_ring=$r) timeout 300 python scripts/time_table.py $A --ops 0 --algos 0 --batches 256 | tail -1; done
for r in 0 9 11 13 16; do echo "== F R ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_ring=$r) timeout 300 python scripts/time_table.py $R --ops 0 --algos 0 --batches 256 | tail -1; done
for r in 0 6 8 10 14; do echo "== BD A ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_bd_ring=$r) timeout 300 python scripts/time_table.py $A --ops 1 --algos 0 --batches 256 | tail -1; done
for r in 0 11 13 16 20; do echo "== BD R ring $r"; UCUDNN_TUNE=$([ $r = 0 ] && echo "" || echo fct_bd_ring=$r) timeout 300 python scripts/time_table.py $R --ops 1 --algos 0 --batches 256 | tail -1; done
