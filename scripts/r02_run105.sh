#!/bin/bash
# TMA implicit GEMM stage-count sweep at the planned micro-batches
for t in "" "pc_stages=4" "pc_stages=6" "pc_ksub=1" "pc_ksub=4"; do
  echo "== $t"
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 --ops 0 --algos 5 --batches 256 | tail -1
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,27,27,192,5,5,2,1 --ops 1 --algos 7 --batches 256 | tail -1
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,384,13,13,256,3,3,1,1 --ops 0 --algos 5 --batches 128 | tail -1
  UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 --ops 0 --algos 5 --batches 64 | tail -1
done
