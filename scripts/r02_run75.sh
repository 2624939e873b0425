#!/bin/bash
# phase_store32: strided BackwardData epilogue decoded per 32-column chunk
timeout 900 python -m pytest tests/test_algos_gpu.py -q -p no:cacheprovider -k "knob and (3-1-2 or ph32 or strip)" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_scale_gpu.py -q -p no:cacheprovider -k "resnet18 and BD" 2>&1 | tail -2
S="256,64,56,56,128,3,3,1,2 256,128,28,28,256,3,3,1,2 256,256,14,14,512,3,3,1,2"
timeout 600 python scripts/time_table.py $S --ops 1 --algos 5 --batches 256,128,64,32
UCUDNN_TUNE=ph32=0 timeout 600 python scripts/time_table.py 256,64,56,56,128,3,3,1,2 --ops 1 --algos 5 --batches 64
