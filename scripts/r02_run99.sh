#!/bin/bash
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob and (2-6 or fct_bf)" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "conv1 and BF" 2>&1 | tail -2
timeout 300 python scripts/time_table.py 256,3,224,224,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 2 --algos 6 --batches 256,128
