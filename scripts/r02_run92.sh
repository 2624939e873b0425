#!/bin/bash
# BackwardFilter TMEM-operand producers: stepped row walk, interior blocks unmasked -- parity + times
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob or 2-6 or bf" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "BF" 2>&1 | tail -2
timeout 600 python scripts/time_table.py 256,3,224,224,64,11,11,2,4 256,3,224,224,64,7,7,3,2 256,64,56,56,64,3,3,1,1 256,128,28,28,128,3,3,1,1 --ops 2 --algos 6 --batches 256
