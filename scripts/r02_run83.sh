#!/bin/bash
# AlexNet BackwardFilter: gather (6) vs channels-last (8) per micro-batch, and the conv2 BF 8@64 launch list
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "a8 or replayed" 2>&1 | tail -2
S="256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1"
timeout 900 python scripts/time_table.py $S --ops 2 --algos 6,8 --batches 256,128,64
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l83.csv python scripts/one_conv.py --layer a2 --op 2 --algo 8 --batch 64 --reps 2 > gpurun_out/l83.out 2>&1
python scripts/launch_times.py gpurun_out/l83.csv; cat gpurun_out/l83.out | tail -2
