#!/bin/bash
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob and fct" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "conv1 and F" 2>&1 | tail -2
timeout 300 python scripts/time_table.py 256,3,224,224,64,7,7,3,2 256,3,224,224,64,11,11,2,4 --ops 0 --algos 0 --batches 256,128
