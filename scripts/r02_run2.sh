#!/bin/bash
# round-2 GPU run 2: zero-workspace implicit GEMM (zgemm) correctness + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_algos_gpu.py tests/test_scale_gpu.py -m gpu -q -p no:cacheprovider --maxfail=30 --timeout 600 -x > gpurun_out/pytest_r2.txt 2>&1
tail -15 gpurun_out/pytest_r2.txt
timeout 600 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1 --algos 0,5,6,8 --batches 256,64 > gpurun_out/tt_r2.txt 2>&1
cat gpurun_out/tt_r2.txt
