#!/bin/bash
# strip kernel: flat tiles across images + faster pad copy -- parity and timings
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "strip or sswap" 2>&1 | tail -3
S="256,64,27,27,192,5,5,2,1 256,64,56,56,64,3,3,1,1"
for t in "strip=1,strip_msub=1" "strip=1,strip_msub=2" "strip=1,strip_msub=4"; do
  echo "== $t"; UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py $S --ops 0,1 --algos 5 --batches 64,32
done
UCUDNN_TUNE=strip=1,strip_msub=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l69a.csv python scripts/one_conv.py --layer a2 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
python scripts/launch_times.py gpurun_out/l69a.csv
UCUDNN_TUNE=strip=1,strip_msub=4,prof=1 timeout 120 python scripts/strip_profile.py 64,64,27,27,192,5,5,2,1 1
UCUDNN_TUNE=strip=1,strip_msub=2,prof=1 timeout 120 python scripts/strip_profile.py 64,64,27,27,192,5,5,2,1 1
