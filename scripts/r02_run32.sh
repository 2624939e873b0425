#!/bin/bash
mkdir -p gpurun_out
for sp in "2 3 31 31 16 11 11 2 4" "2 3 36 36 70 7 7 3 2" "3 3 227 227 64 11 11 0 4" "2 3 224 224 64 7 7 3 2" "1 2 40 40 8 11 11 0 4" "3 4 30 30 24 5 5 2 2" "5 3 63 63 20 11 11 1 4" "4 3 48 48 64 7 7 3 2" "2 1 20 20 5 3 3 1 2"; do
  timeout 60 python scripts/one_small.py $sp 2 6 2>&1 | tail -2
done
timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256,64
UCUDNN_TUNE=fct_bf=0 timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256
