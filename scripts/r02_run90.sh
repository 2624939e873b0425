#!/bin/bash
# ResNet-50 strided 1x1 BackwardFilter / Forward: algorithms and CTA pairs
S="256,256,56,56,512,1,1,0,2 256,1024,14,14,2048,1,1,0,2 256,512,28,28,1024,1,1,0,2"
timeout 900 python scripts/time_table.py $S --ops 0,2 --algos 0,3,5,6,7,8 --batches 256,128,64
echo "== bfn2=1"; UCUDNN_TUNE=bfn2=1 timeout 600 python scripts/time_table.py $S --ops 2 --algos 8 --batches 256,128,64
S1="256,256,56,56,64,1,1,0,1 256,64,56,56,256,1,1,0,1 256,1024,14,14,256,1,1,0,1 256,256,14,14,1024,1,1,0,1"
echo "== 1x1 s1 default"; timeout 600 python scripts/time_table.py $S1 --ops 2 --algos 0,6,8 --batches 256,128
echo "== 1x1 s1 bfn2=1"; UCUDNN_TUNE=bfn2=1 timeout 600 python scripts/time_table.py $S1 --ops 2 --algos 8 --batches 256,128
