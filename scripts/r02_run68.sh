#!/bin/bash
# launch list of conv2 BD through the strip kernel (64 images) and the planned sliced kernel (256)
UCUDNN_TUNE=strip=1,strip_msub=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l68a.csv python scripts/one_conv.py --layer a2 --op 1 --algo 5 --batch 64 --reps 2 > /dev/null 2>&1
python scripts/launch_times.py gpurun_out/l68a.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l68b.csv python scripts/one_conv.py --layer a2 --op 1 --algo 7 --batch 256 --reps 2 > /dev/null 2>&1
python scripts/launch_times.py gpurun_out/l68b.csv
