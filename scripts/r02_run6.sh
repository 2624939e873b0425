#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_algos_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -k "knob or [0-" > gpurun_out/pytest_r6a.txt 2>&1
tail -3 gpurun_out/pytest_r6a.txt
timeout 900 python -m pytest tests/test_scale_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_r6b.txt 2>&1
tail -3 gpurun_out/pytest_r6b.txt
L="256,3,227,227,64,11,11,2,4 256,64,27,27,192,5,5,2,1 256,192,13,13,384,3,3,1,1 256,384,13,13,256,3,3,1,1 256,256,13,13,256,3,3,1,1"
timeout 600 python scripts/time_table.py $L --ops 0,1,2 --algos 0 --batches 256 > gpurun_out/tt_r6.txt 2>&1
cat gpurun_out/tt_r6.txt
rm -f gpurun_out/db6.csv
timeout 900 python bench.py --steps 20 --warmup 5 --db gpurun_out/db6.csv > gpurun_out/bench6.json 2> gpurun_out/bench6.err
cat gpurun_out/bench6.json
