#!/bin/bash
# fct_bwdd producer / issuer without runtime divisions: parity + times
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "fct_bd or (knob and 1-0])" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -x -k "not knob and not bf" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "(resnet18 and conv1 and BD) or (alexnet_algorithm_at_scale and conv1-BD)" 2>&1 | tail -2
timeout 600 python scripts/time_table.py 256,3,224,224,64,7,7,3,2 256,3,224,224,64,11,11,2,4 --ops 1 --algos 0 --batches 256,128,64
