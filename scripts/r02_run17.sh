#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "[0-" > gpurun_out/pytest_r17a.txt 2>&1
tail -3 gpurun_out/pytest_r17a.txt
L="256,64,56,56,64,1,1,0,1 256,64,56,56,256,1,1,0,1 256,256,56,56,64,1,1,0,1 256,512,28,28,128,1,1,0,1 256,1024,14,14,256,1,1,0,1"
timeout 600 python scripts/time_table.py $L --ops 0,1 --algos 0 --batches 256 > gpurun_out/tt_r17.txt 2>&1
cat gpurun_out/tt_r17.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:z1x1 -s 1 -c 1 -o gpurun_out/r02_z1x1_res2_f python scripts/one_conv.py --shape 256,64,56,56,256,1,1,0,1 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
