#!/bin/bash
timeout 900 python -m pytest tests/test_algos_gpu.py tests/test_deterministic_gpu.py -m gpu -q -p no:cacheprovider --timeout 600 -x -k "BF or bf or determin or knob" 2>&1 | tail -2
timeout 120 python scripts/time_table.py 256,3,227,227,64,11,11,0,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256,64
