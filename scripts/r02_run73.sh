#!/bin/bash
# ResNet-18 strided 3x3 BackwardData: per-algorithm times and launch lists
S="256,64,56,56,128,3,3,1,2 256,128,28,28,256,3,3,1,2 256,256,14,14,512,3,3,1,2"
UCUDNN_TUNE=trace=1 timeout 600 python scripts/time_table.py $S --ops 1 --algos 0,3,5,7,8 --batches 256,128,64,32
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l73a.csv python scripts/one_conv.py --shape 256,64,56,56,128,3,3,1,2 --op 1 --algo 0 --batch 256 --reps 2 > gpurun_out/l73a.out 2>&1
python scripts/launch_times.py gpurun_out/l73a.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l73b.csv python scripts/one_conv.py --shape 256,64,56,56,128,3,3,1,2 --op 1 --algo 5 --batch 64 --reps 2 > gpurun_out/l73b.out 2>&1
python scripts/launch_times.py gpurun_out/l73b.csv
python scripts/one_small.py 2 64 16 16 128 3 3 1 2 1 0 | grep trace
python scripts/one_small.py 2 64 16 16 128 3 3 1 2 1 5 | grep trace
