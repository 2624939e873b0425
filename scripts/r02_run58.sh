#!/bin/bash
for sp in "2 64 56 56 128 1 1 0 2" "3 32 28 28 64 1 1 0 2" "2 48 14 14 96 1 1 0 2" "2 64 15 15 32 1 1 0 2" "2 16 20 20 24 1 1 0 3"; do
  timeout 60 python scripts/one_small.py $sp 0 5 2>&1 | grep -E "exact|rror|trace"
done
timeout 200 python scripts/time_table.py 256,256,56,56,512,1,1,0,2 256,512,28,28,1024,1,1,0,2 256,1024,14,14,2048,1,1,0,2 --ops 0 --algos 0,5 --batches 256,128,64 2>&1
UCUDNN_TUNE=pc_subsample=0 timeout 200 python scripts/time_table.py 256,256,56,56,512,1,1,0,2 256,512,28,28,1024,1,1,0,2 --ops 0 --algos 5 --batches 256,64 2>&1
