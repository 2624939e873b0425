#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "BF and 6" -x > gpurun_out/pytest_r8a.txt 2>&1
tail -3 gpurun_out/pytest_r8a.txt
timeout 300 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256 > gpurun_out/tt_r8.txt 2>&1
cat gpurun_out/tt_r8.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bfs_kernel -s 1 -c 1 -o gpurun_out/r02_bfs2_conv1_bf python scripts/one_conv.py --shape 256,3,227,227,64,11,11,2,4 --op 2 --algo 6 --batch 256 --reps 2 > /dev/null 2>&1
ls gpurun_out | grep bfs2
