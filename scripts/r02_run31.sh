#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -x -k "5 or 7" > gpurun_out/pytest_r31.txt 2>&1
tail -3 gpurun_out/pytest_r31.txt
L="256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1 256,128,28,28,128,3,3,1,1 256,256,14,14,256,3,3,1,1 256,64,56,56,64,3,3,1,1"
timeout 300 python scripts/time_table.py $L --ops 0,1 --algos 5 --batches 256,64 2>&1
