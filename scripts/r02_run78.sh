#!/bin/bash
# ResNet conv1 BackwardData (7x7 stride 2, 3 channels) through algorithm 0 at 256 images
timeout 300 python scripts/one_conv.py --shape 256,3,224,224,64,7,7,3,2 --op 1 --algo 0 --batch 256 --reps 1 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fct -s 1 -c 1 \
  -o gpurun_out/fct_bwdd_r50conv1 python scripts/one_conv.py --shape 256,3,224,224,64,7,7,3,2 --op 1 --algo 0 --batch 256 --reps 2 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/fct_bwdd_r50conv1.ncu-rep
