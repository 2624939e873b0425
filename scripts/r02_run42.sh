#!/bin/bash
for t in "strip_msub=2" "strip_msub=4" "strip_msub=4,strip_nsb=2" "strip_msub=3"; do
  UCUDNN_TUNE=strip=1,prof=1,$t timeout 60 python scripts/strip_profile.py 256,64,27,27,192,5,5,2,1 1 2>&1 | tail -1
  UCUDNN_TUNE=strip=1,prof=1,$t timeout 60 python scripts/strip_profile.py 256,64,56,56,64,3,3,1,1 1 2>&1 | tail -1
done
for t in "strip=1,strip_msub=4" "strip=1,strip_msub=3"; do
for sp in "2 64 27 27 96 5 5 2 1 1 5" "3 32 14 14 64 3 3 1 1 0 5" "5 64 27 27 192 5 5 2 1 1 5" "2 96 11 9 48 3 3 1 1 0 5"; do
  UCUDNN_TUNE=$t timeout 60 python scripts/one_small.py $sp 2>&1 | grep -E "exact|rror|trace"
done
done
