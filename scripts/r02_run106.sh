#!/bin/bash
# pc_ksub=1 across the planned TMA implicit GEMM calls
for t in "" "pc_ksub=1"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,128,28,28,128,3,3,1,1 --ops 0,1 --algos 5 --batches 128 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,192,13,13,384,3,3,1,1 --ops 0 --algos 5 --batches 256 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,192,13,13,384,3,3,1,1 --ops 1 --algos 7 --batches 256 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,256,13,13,256,3,3,1,1 --ops 0,1 --algos 5 --batches 256 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,384,13,13,256,3,3,1,1 --ops 1 --algos 5 --batches 256 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 --ops 1 --algos 5 --batches 64 | grep algo
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,56,56,128,3,3,1,2 256,128,28,28,256,3,3,1,2 --ops 1 --algos 5 --batches 128 | grep algo
done
