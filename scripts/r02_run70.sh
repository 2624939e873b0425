#!/bin/bash
# strip kernel: double strip buffers with fewer filter stages at 4 sub-tiles
S="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1"
for t in "strip=1,strip_msub=4" "strip=1,strip_msub=4,strip_minst=3" "strip=1,strip_msub=4,strip_minst=2" "strip=1,strip_msub=2,strip_minst=3"; do
  echo "== $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $S --ops 0,1 --algos 5 --batches 64,32
done
for t in "strip=1,strip_msub=4,strip_minst=3,prof=1" "strip=1,strip_msub=4,strip_minst=2,prof=1"; do
UCUDNN_TUNE=$t timeout 120 python scripts/strip_profile.py 64,64,27,27,192,5,5,2,1 1
UCUDNN_TUNE=$t timeout 120 python scripts/strip_profile.py 64,64,56,56,64,3,3,1,1 1
done
UCUDNN_TUNE=strip=1,strip_msub=4,strip_minst=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l70a.csv python scripts/one_conv.py --shape 64,64,56,56,64,3,3,1,1 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
python scripts/launch_times.py gpurun_out/l70a.csv
