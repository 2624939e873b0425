#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "[0-" > gpurun_out/pytest_r24.txt 2>&1
tail -2 gpurun_out/pytest_r24.txt
timeout 900 python -m pytest tests/test_scale_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "a0 or zz" > gpurun_out/pytest_r24b.txt 2>&1
tail -2 gpurun_out/pytest_r24b.txt
L="256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 256,64,56,56,64,3,3,1,1 256,64,27,27,192,5,5,2,1"
timeout 600 python scripts/time_table.py $L --ops 1 --algos 0,5 --batches 256 > gpurun_out/tt_r24.txt 2>&1
UCUDNN_TUNE=z_bres=0 timeout 600 python scripts/time_table.py $L --ops 1 --algos 0 --batches 256 >> gpurun_out/tt_r24.txt 2>&1
cat gpurun_out/tt_r24.txt
