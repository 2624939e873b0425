#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider -x --timeout 600 -k "knob or [0-" > gpurun_out/pytest_r4.txt 2>&1
tail -3 gpurun_out/pytest_r4.txt
timeout 600 python scripts/time_table.py 256,3,227,227,64,11,11,2,4 256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 --ops 0,1 --algos 0 --batches 256 > gpurun_out/tt_r4.txt 2>&1
cat gpurun_out/tt_r4.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 1 -c 1 \
  -o gpurun_out/r02_zgemm16_conv2_f python scripts/one_conv.py --layer a2 --op 0 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
ls gpurun_out
