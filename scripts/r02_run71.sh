#!/bin/bash
for sh in 64,64,27,27,192,5,5,2,1 64,64,56,56,64,3,3,1,1; do
UCUDNN_TUNE=strip=1,strip_msub=4,strip_minst=3,prof=1 timeout 120 python scripts/strip_profile.py $sh 1
UCUDNN_TUNE=strip=1,strip_msub=4,strip_minst=3,prof=2 timeout 120 python scripts/strip_profile.py $sh 1
done
