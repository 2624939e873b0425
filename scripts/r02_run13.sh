#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "0-F" -x > gpurun_out/pytest_r13a.txt 2>&1
tail -1 gpurun_out/pytest_r13a.txt
timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 0 --algos 0 --batches 256,64 > gpurun_out/tt_r13.txt 2>&1
for t in fps_stages=2 fps_stages=3; do UCUDNN_TUNE=$t timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 --ops 0 --algos 0 --batches 256 >> gpurun_out/tt_r13.txt 2>&1; done
cat gpurun_out/tt_r13.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fps_kernel -s 1 -c 1 -o gpurun_out/r02_fps2_conv1_f python scripts/one_conv.py --shape 256,3,227,227,64,11,11,2,4 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
