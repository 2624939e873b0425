#!/bin/bash
# strip implicit GEMM on the narrow-N stride-1 shapes: msub / nsb sweep + MMA-warp wait split
S="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1"
echo "== default"; timeout 300 python scripts/time_table.py $S --ops 0,1 --algos 5,7 --batches 64,32
for t in "strip=1,strip_msub=1" "strip=1,strip_msub=2" "strip=1,strip_msub=4" "strip=1,strip_msub=4,strip_nsb=2" "strip=1,strip_msub=2,strip_nsb=2"; do
  echo "== $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $S --ops 0,1 --algos 5 --batches 64,32
done
for t in "strip=1,strip_msub=2,prof=1" "strip=1,strip_msub=4,prof=1" "strip=1,strip_msub=4,strip_nsb=2,prof=1"; do
  UCUDNN_TUNE=$t timeout 120 python scripts/strip_profile.py 64,64,27,27,192,5,5,2,1 1
  UCUDNN_TUNE=$t timeout 120 python scripts/strip_profile.py 64,64,56,56,64,3,3,1,1 1
done
