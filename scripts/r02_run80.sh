#!/bin/bash
# RingPos in the fct kernels' producer / issuer loops: parity + times
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -x -k "not knob" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "resnet18 or conv1" 2>&1 | tail -2
timeout 600 python scripts/time_table.py 256,3,224,224,64,11,11,2,4 256,3,224,224,64,7,7,3,2 --ops 0,1,2 --algos 0,6 --batches 256
timeout 600 python scripts/time_table.py 256,64,56,56,64,3,3,1,1 --ops 2 --algos 6 --batches 256
